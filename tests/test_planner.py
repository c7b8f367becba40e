"""CPU tests of the roofline planner / autotuner host logic (planner.py) against
hand-computed values of the paper's formulas."""
import math

import pytest

from paper_1809_07851_b200 import planner


def _info(nk1_b, nk2_b, nk3_b, nk3_f, nk4_b):
    return {"alg_bytes": [nk1_b, nk2_b, nk3_b, nk4_b], "alg_flops": [0.0, 0.0, nk3_f, 0.0]}


def test_stage_sum_model_hand_values():
    # MB = 1000 GB/s, Peak = 10 TFLOP/s: stage times max(F/P, DM/MB)
    info = _info(1e9, 2e9, 1e9, 50e12, 3e9)
    st = planner.predict_stage_seconds(info, 1000.0, 10.0)
    assert st == pytest.approx([1e-3, 2e-3, 5.0, 3e-3])  # NK3 compute-bound: 50e12 / 10e12
    info2 = _info(1e9, 2e9, 8e9, 1e10, 3e9)              # NK3 memory-bound: 8e9 / 1e12 > 1e10 / 1e13
    assert planner.predict_seconds(info2, 1000.0, 10.0) == pytest.approx(1e-3 + 2e-3 + 8e-3 + 3e-3)


def test_best_m_ties_to_smaller_m_and_speedup_definition():
    times = {("winograd", 2): 3.0, ("winograd", 4): 2.0, ("winograd", 6): 2.0,
             ("regular_fft", 8): 1.5, ("regular_fft", 14): 1.0, ("gauss_fft", 14): 4.0}
    b = planner.best_m(times)
    assert b["winograd"] == (4, 2.0)          # tie between m=4 and m=6 -> smaller m
    assert b["regular_fft"] == (14, 1.0)
    sp = planner.speedups(b)
    # Speedup(A, B) = T_B / T_A: FFT twice as fast -> 2.0
    assert sp["regular_fft_vs_winograd"] == pytest.approx(2.0)
    assert sp["gauss_fft_vs_winograd"] == pytest.approx(0.5)


def test_rrmse_and_fitness():
    assert planner.rrmse([1.1, 0.9], [1.0, 1.0]) == pytest.approx(0.1)
    assert planner.fitness(0.0) == 100.0
    # the paper's pair: rRMSE 0.079 -> fitness 92.68 %
    assert planner.fitness(0.079) == pytest.approx(92.68, abs=0.01)
    assert planner.fitness(0.1) == pytest.approx(90.9, abs=0.05)
    with pytest.raises(ValueError):
        planner.rrmse([], [])


def test_report_on_real_plan_geometry():
    import paper_1809_07851_b200 as fc
    from paper_1809_07851_b200 import _build
    _build.build()
    infos = {(meth, m): fc.plan_query(64, 256, 256, 58, 58, 3, meth, m)
             for meth, m in (("winograd", 4), ("winograd", 6), ("regular_fft", 14), ("gauss_fft", 14))}
    meas = {k: 1.0 for k in infos}
    rep = planner.report(infos, meas, 6555.8, 274.15)
    # Winograd F(4,3) on VGG-3.2: NK3 59.2 GFLOP at 274 TFLOP/s dominates its stage
    t_w4 = rep["predicted_ms"]["winograd/m=4"]
    assert 0.3 < t_w4 < 0.6
    assert rep["best_m_measured"]["winograd"] == 4
    assert "speedup_rrmse" in rep and math.isfinite(rep["speedup_fitness"])

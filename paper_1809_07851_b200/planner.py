"""Roofline planner and tile-size autotuner -- host logic only.

The paper estimates a layer's running time by its stage-sum roofline model
(Eq. "running time" and "running time_total"):

    T_total = sum_s FPO_s / MB / min(CMR, AI_s) = sum_s max(FPO_s / Peak, DM_s / MB)

and compares methods at the m that minimises each method's running time
(Eq. eq_new_speedup), with Speedup(A, B) = T_B / T_A
(P:784-796).  The model's agreement with measurement is reported as the
relative RMSE of the predicted vs measured speedups and fitness =
100 / (1 + rRMSE).

Here the machine is one B200: MB = measured HBM copy bandwidth, the contraction's
Peak = the tensor-core fp32-equivalent peak of the 3xTF32 split (TF32 peak / 3),
and the transforms are charged their HBM bytes (their FLOP counts come from the
paper's genfft/wincnn tables, whose AIs <= 6.9 sit far below B200's CMR, P:872-882,
so FPO/Peak never binds).  Per-stage FPO/DM are the plan's algorithmic
counts (conv_plan_info.alg_bytes / alg_flops, Table layer-stuff).
"""
from __future__ import annotations

import math

STAGES = ("NK1 kernel transform", "NK2 input transform", "NK3 contraction", "NK4 output transform")


def predict_stage_seconds(info: dict, hbm_gbs: float, contraction_tflops: float) -> list[float]:
    """Per-stage roofline time max(FPO/Peak, DM/MB) in seconds."""
    out = []
    for s in range(4):
        t_mem = info["alg_bytes"][s] / (hbm_gbs * 1e9)
        t_cmp = info["alg_flops"][s] / (contraction_tflops * 1e12) if s == 2 else 0.0
        out.append(max(t_mem, t_cmp))
    return out


def predict_seconds(info: dict, hbm_gbs: float, contraction_tflops: float) -> float:
    """Stage-sum model T_total."""
    return sum(predict_stage_seconds(info, hbm_gbs, contraction_tflops))


def best_m(times: dict) -> dict:
    """times: {(method, m): seconds} -> {method: (m, seconds)} at each method's fastest m;
    ties go to the smaller m."""
    best = {}
    for (method, m), t in sorted(times.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        if method not in best or t < best[method][1]:
            best[method] = (m, t)
    return best


def speedups(best: dict, base: str = "winograd") -> dict:
    """Speedup(A, base) = T_base / T_A at each method's best m (Eq. eq_new_speedup)."""
    if base not in best:
        return {}
    tb = best[base][1]
    return {"%s_vs_%s" % (meth, base): tb / t for meth, (m, t) in best.items() if meth != base}


def rrmse(pred: list[float], meas: list[float]) -> float:
    """Relative root-mean-square error of predictions against measurements."""
    if not pred or len(pred) != len(meas):
        raise ValueError("need equal, non-empty lists")
    return math.sqrt(sum(((p - q) / q) ** 2 for p, q in zip(pred, meas)) / len(pred))


def fitness(r: float) -> float:
    """fitness = 100 / (1 + rRMSE) (P:850-852 footnote)."""
    return 100.0 / (1.0 + r)


def report(infos: dict, measured_ms: dict, hbm_gbs: float, contraction_tflops: float) -> dict:
    """Model vs measurement over one layer's (method, m) sweep.

    infos: {(method, m): conv_plan_info dict}; measured_ms: {(method, m): ms}.
    Returns predicted ms, the model's and the measurement's best m per method, the
    predicted and measured speedups over Winograd, and rRMSE / fitness of the
    speedups (the paper's accuracy measure) and of the absolute times."""
    pred = {k: predict_seconds(v, hbm_gbs, contraction_tflops) for k, v in infos.items()}
    meas = {k: v * 1e-3 for k, v in measured_ms.items() if k in pred}
    bp, bm = best_m(pred), best_m(meas)
    sp, sm = speedups(bp), speedups(bm)
    keys = sorted(set(sp) & set(sm))
    out = {
        "model": "stage-sum roofline (P:772-780), MB=%.0f GB/s, contraction peak=%.1f TFLOP/s"
                 % (hbm_gbs, contraction_tflops),
        "predicted_ms": {"%s/m=%d" % k: round(v * 1e3, 4) for k, v in sorted(pred.items())},
        "best_m_model": {k: v[0] for k, v in bp.items()},
        "best_m_measured": {k: v[0] for k, v in bm.items()},
        "speedup_model": sp,
        "speedup_measured": sm,
        "efficiency": {"%s/m=%d" % k: round(pred[k] / meas[k], 4) for k in sorted(meas)},
    }
    if keys:
        r = rrmse([sp[k] for k in keys], [sm[k] for k in keys])
        out["speedup_rrmse"] = r
        out["speedup_fitness"] = fitness(r)
    return out

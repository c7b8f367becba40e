"""The fp32 multithreaded CPU direct convolution bench.py times as a baseline agrees with
the fp64 oracle to fp32 accumulation accuracy (it is a baseline, not a parity reference)."""
import numpy as np

import cpu_baseline
import oracle
import synth


def test_cpu_direct_fp32_matches_oracle():
    for cfg in (synth.custom(2, 7, 5, 13, 11, 3, seed=3), synth.custom(1, 16, 8, 20, 20, 5, seed=4, dist="normal")):
        I, W = synth.make_inputs(cfg)
        O = oracle.conv_fp64(I, W)
        y = cpu_baseline.conv_fp32(I, W).astype(np.float64)
        assert y.shape == O.shape
        assert np.abs(y - O).max() / np.abs(O).max() < 1e-5
    assert cpu_baseline.num_threads() >= 1

"""Pins for oracle/ (CPU only): the oracle is checked against things other than itself.

* hand-computed cases (tests/golden/hand_cases.json, each cited);
* math.fsum brute force of the exact fp64 products at sampled outputs;
* torch.nn.functional.conv2d in float64 on CPU (an independent library
  cross-correlation routine);
* invariants on integer-valued data (where every fp64 sum is exact, so they
  must hold bit-exactly): linearity, delta kernel = shifted input, shift
  equivariance, C-additivity, zero weights, batch independence, output-channel
  permutation.

A dropped term, wrong sign, flipped kernel, swapped c/c' index or off-by-one
bound in oracle/conv_oracle.c fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")


def _int_data(shape, seed, lo=-8, hi=8):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, size=shape).astype(np.float32)


def test_hand_cases():
    cases = json.load(open(GOLDEN))["cases"]
    assert len(cases) >= 5
    for case in cases:
        I = np.asarray(case["I"], dtype=np.float32)
        W = np.asarray(case["W"], dtype=np.float32)
        O = oracle.conv_fp64(I, W)
        np.testing.assert_array_equal(O, np.asarray(case["O"], dtype=np.float64), err_msg=case["name"])


def test_flipped_kernel_differs():
    # true convolution (kernel flip) would give [[23,33],[53,63]] for the orientation case
    I = np.arange(1, 10, dtype=np.float32).reshape(1, 1, 3, 3)
    W = np.array([[[[1, 2], [3, 4]]]], dtype=np.float32)
    O = oracle.conv_fp64(I, W)
    assert not np.array_equal(O[0, 0], np.array([[23, 33], [53, 63]], dtype=np.float64))


@pytest.mark.parametrize("shape", [(2, 5, 3, 9, 11, 3), (1, 7, 2, 12, 8, 5), (3, 2, 4, 6, 6, 1)])
def test_fsum_bruteforce(shape):
    B, C, Co, H, Wd, r = shape
    g = torch.Generator().manual_seed(7)
    I = (torch.rand(B, C, H, Wd, generator=g) * 2 - 1).numpy()
    W = (torch.rand(Co, C, r, r, generator=g) * 2 - 1).numpy()
    O = oracle.conv_fp64(I, W)
    Ho, Wo = H - r + 1, Wd - r + 1
    rng = np.random.default_rng(3)
    for _ in range(60):
        b, co, i, j = rng.integers(B), rng.integers(Co), rng.integers(Ho), rng.integers(Wo)
        terms = [float(I[b, c, i + p, j + q]) * float(W[co, c, p, q])
                 for c in range(C) for p in range(r) for q in range(r)]
        exact = math.fsum(terms)  # correctly rounded exact sum (products are exact in fp64)
        scale = max(abs(t) for t in terms) or 1.0
        assert abs(O[b, co, i, j] - exact) <= 1e-13 * scale * len(terms)
    # corners too (ragged borders)
    for (i, j) in ((0, 0), (0, Wo - 1), (Ho - 1, 0), (Ho - 1, Wo - 1)):
        terms = [float(I[B - 1, c, i + p, j + q]) * float(W[Co - 1, c, p, q])
                 for c in range(C) for p in range(r) for q in range(r)]
        assert abs(O[B - 1, Co - 1, i, j] - math.fsum(terms)) <= 1e-13 * len(terms)


def test_sampled_equals_full():
    cfg = synth.custom(2, 6, 5, 13, 10, 3, seed=11)
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    idx = synth.sample_output_indices(cfg, 200, seed=5)
    s = oracle.conv_fp64_sampled(I, W, idx)
    np.testing.assert_array_equal(s, O[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]])


@pytest.mark.parametrize("name", ["tiny", "small_r5", "rect"])
def test_torch_conv2d_fp64(name):
    cfg = {"tiny": synth.CONFIGS["tiny"],
           "small_r5": synth.custom(2, 8, 6, 20, 20, 5, seed=3, dist="normal"),
           "rect": synth.custom(3, 5, 7, 17, 29, 3, seed=4)}[name]
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    ref = torch.nn.functional.conv2d(I.double(), W.double()).numpy()
    assert O.shape == ref.shape
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


def test_linearity_exact():
    I1 = _int_data((2, 3, 10, 9), 1)
    I2 = _int_data((2, 3, 10, 9), 2)
    W1 = _int_data((4, 3, 3, 3), 3)
    W2 = _int_data((4, 3, 3, 3), 4)
    a = np.float32(3.0)
    np.testing.assert_array_equal(oracle.conv_fp64(a * I1 + I2, W1),
                                  3.0 * oracle.conv_fp64(I1, W1) + oracle.conv_fp64(I2, W1))
    np.testing.assert_array_equal(oracle.conv_fp64(I1, a * W1 + W2),
                                  3.0 * oracle.conv_fp64(I1, W1) + oracle.conv_fp64(I1, W2))


@pytest.mark.parametrize("r,p0,q0", [(3, 0, 0), (3, 1, 2), (5, 4, 1), (2, 1, 1)])
def test_delta_kernel_shifts_input(r, p0, q0):
    C = 4
    I = np.random.default_rng(9).standard_normal((2, C, 12, 11)).astype(np.float32)
    W = np.zeros((C, C, r, r), dtype=np.float32)
    for c in range(C):
        W[c, c, p0, q0] = 1.0
    O = oracle.conv_fp64(I, W)
    Ho, Wo = 12 - r + 1, 11 - r + 1
    np.testing.assert_array_equal(O, I[:, :, p0:p0 + Ho, q0:q0 + Wo].astype(np.float64))


def test_shift_equivariance():
    I = _int_data((1, 3, 16, 16), 5)
    W = _int_data((2, 3, 3, 3), 6)
    dy, dx = 2, 3
    Is = np.zeros_like(I)
    Is[:, :, dy:, dx:] = I[:, :, :16 - dy, :16 - dx]
    O = oracle.conv_fp64(I, W)
    Os = oracle.conv_fp64(Is, W)
    # output of shifted input, shifted back, equals the original on the overlap
    np.testing.assert_array_equal(Os[:, :, dy:, dx:], O[:, :, :14 - dy, :14 - dx])


def test_c_additivity_zero_batch_permutation():
    I = _int_data((3, 6, 9, 9), 7)
    W = _int_data((5, 6, 3, 3), 8)
    O = oracle.conv_fp64(I, W)
    np.testing.assert_array_equal(
        O, oracle.conv_fp64(I[:, :2].copy(), W[:, :2].copy()) + oracle.conv_fp64(I[:, 2:].copy(), W[:, 2:].copy()))
    np.testing.assert_array_equal(oracle.conv_fp64(I, np.zeros_like(W)), np.zeros_like(O))
    for b in range(3):
        np.testing.assert_array_equal(O[b:b + 1], oracle.conv_fp64(I[b:b + 1].copy(), W))
    perm = np.array([3, 0, 4, 1, 2])
    np.testing.assert_array_equal(oracle.conv_fp64(I, W[perm].copy()), O[:, perm])


def test_rejects_bad_shapes():
    with pytest.raises(ValueError):
        oracle.conv_fp64(np.zeros((1, 1, 2, 2), np.float32), np.zeros((1, 1, 3, 3), np.float32))
    with pytest.raises(TypeError):
        oracle.conv_fp64(np.zeros((1, 1, 4, 4), np.float64), np.zeros((1, 1, 3, 3), np.float32))
    cfg = synth.custom(1, 1, 1, 5, 5, 3)
    I, W = synth.make_inputs(cfg)
    with pytest.raises(ValueError):
        oracle.conv_fp64_sampled(I, W, [[0, 0, 3, 0]])


# ------------------------------------------------------------ N-D oracle ---
# oracle.conv_nd_fp64 (P:926-929 N-dimensional / non-isotropic extension of Eq. 5)

@pytest.mark.parametrize("ishape,wshape", [((2, 3, 17), (4, 3, 5)), ((2, 3, 9, 11, 8), (2, 3, 3, 2, 4)),
                                           ((1, 2, 6, 5, 7), (3, 2, 1, 3, 2))])
def test_nd_against_torch_convnd(ishape, wshape):
    """torch's float64 conv1d / conv3d on CPU (an independent library routine)."""
    g = torch.Generator().manual_seed(7)
    I = torch.randn(ishape, generator=g)
    W = torch.randn(wshape, generator=g)
    O = oracle.conv_nd_fp64(I, W)
    f = {3: torch.nn.functional.conv1d, 5: torch.nn.functional.conv3d}[len(ishape)]
    R = f(I.double(), W.double()).numpy()
    assert O.shape == R.shape
    assert np.abs(O - R).max() <= 1e-12 * np.abs(R).max()


def test_nd_fsum_bruteforce():
    """Every fp32 product is exact in fp64: math.fsum of the products at sampled 3-D outputs
    is the correctly rounded exact sum."""
    rng = np.random.default_rng(3)
    I = rng.standard_normal((2, 3, 7, 6, 9)).astype(np.float32)
    W = rng.standard_normal((2, 3, 3, 2, 4)).astype(np.float32)
    O = oracle.conv_nd_fp64(I, W)
    for _ in range(64):
        b, co = rng.integers(0, 2), rng.integers(0, 2)
        i0, i1, i2 = rng.integers(0, 5), rng.integers(0, 5), rng.integers(0, 6)
        terms = [float(I[b, c, i0 + p, i1 + q, i2 + s]) * float(W[co, c, p, q, s])
                 for c in range(3) for p in range(3) for q in range(2) for s in range(4)]
        assert abs(O[b, co, i0, i1, i2] - math.fsum(terms)) <= 1e-13 * max(1.0, max(abs(x) for x in terms))


@pytest.mark.parametrize("tap", [(0, 0, 0), (1, 2, 0), (2, 0, 3)])
def test_nd_delta_kernel_shifts_input(tap):
    """W[c'][c] = delta_{c'c} delta_{p, tap}: O[b][c] is I[b][c] shifted by tap, exactly."""
    I = _int_data((2, 3, 6, 7, 8), 11)
    W = np.zeros((3, 3, 3, 3, 4), dtype=np.float32)
    for c in range(3):
        W[c, c][tap] = 1.0
    O = oracle.conv_nd_fp64(I, W)
    a, b_, c_ = tap
    assert np.array_equal(O, I[:, :, a:a + 4, b_:b_ + 5, c_:c_ + 5].astype(np.float64))


def test_nd_separable_kernel_closed_form():
    """A rank-one kernel W = u (x) v (x) w (C = C' = 1) convolves axis by axis: three
    successive 1-D valid correlations (numpy.correlate), exact on integer data."""
    I = _int_data((1, 1, 7, 6, 9), 12)
    u, v, w = np.array([1, -2, 3], np.float32), np.array([2, 1], np.float32), np.array([-1, 0, 2, 1], np.float32)
    W = np.einsum("i,j,k->ijk", u, v, w).astype(np.float32)[None, None]
    O = oracle.conv_nd_fp64(I, W)[0, 0]
    x = I[0, 0].astype(np.float64)
    x = np.apply_along_axis(lambda a: np.correlate(a, w, "valid"), 2, x)
    x = np.apply_along_axis(lambda a: np.correlate(a, v, "valid"), 1, x)
    x = np.apply_along_axis(lambda a: np.correlate(a, u, "valid"), 0, x)
    assert np.array_equal(O, x)


def test_nd_two_d_matches_the_2d_oracle():
    """nd = 2 with a square kernel is Eq. 5 itself: bit-identical to oracle.conv_fp64 (same
    (c, p, q) summation order), and a 1 x r kernel is the 1-D correlation of every row."""
    I, W = synth.make_inputs(synth.custom(2, 3, 4, 9, 11, 3, seed=13, dist="normal"))
    assert np.array_equal(oracle.conv_nd_fp64(I, W), oracle.conv_fp64(I, W))
    I1 = _int_data((1, 1, 4, 9), 14)
    k = np.array([3, -1, 2], np.float32)
    O = oracle.conv_nd_fp64(I1, k.reshape(1, 1, 1, 3))[0, 0]
    assert np.array_equal(O, np.stack([np.correlate(row.astype(np.float64), k, "valid") for row in I1[0, 0]]))


def test_nd_rejects_bad_shapes():
    with pytest.raises(ValueError):
        oracle.conv_nd_fp64(np.zeros((1, 2, 3, 3, 3, 3), np.float32), np.zeros((1, 2, 1, 1, 1, 1), np.float32))
    with pytest.raises(ValueError):
        oracle.conv_nd_fp64(np.zeros((1, 2, 3), np.float32), np.zeros((1, 2, 4), np.float32))


# ----------------------------------------------------------- gradients ---
# oracle.conv_bwd_data_fp64 / conv_bwd_filter_fp64 (the adjoints of Eq. 5, written out)

def test_backward_adjoint_identities_exact():
    """<conv(I, W), dY> = <I, bwd_data(dY, W)> = <W, bwd_filter(I, dY)>, exactly on integer data
    (every fp64 sum exact): a transposed or shifted index in either gradient breaks it."""
    I = _int_data((2, 3, 7, 8), 21, -3, 3)
    W = _int_data((4, 3, 3, 3), 22, -3, 3)
    dY = _int_data((2, 4, 5, 6), 23, -3, 3)
    O = oracle.conv_fp64(I, W)
    lhs = float(np.sum(O * dY))
    dX = oracle.conv_bwd_data_fp64(dY, W, 7, 8)
    dW = oracle.conv_bwd_filter_fp64(I, dY, 3)
    assert lhs == float(np.sum(I.astype(np.float64) * dX)) == float(np.sum(W.astype(np.float64) * dW))


def test_backward_against_torch_autograd_fp64():
    """torch.nn.grad.conv2d_input / conv2d_weight in float64 on CPU (library routines)."""
    g = torch.Generator().manual_seed(5)
    I = torch.randn(2, 3, 9, 10, generator=g)
    W = torch.randn(4, 3, 3, 3, generator=g)
    dY = torch.randn(2, 4, 7, 8, generator=g)
    dX = oracle.conv_bwd_data_fp64(dY, W, 9, 10)
    dW = oracle.conv_bwd_filter_fp64(I, dY, 3)
    rx = torch.nn.grad.conv2d_input(I.shape, W.double(), dY.double()).numpy()
    rw = torch.nn.grad.conv2d_weight(I.double(), W.shape, dY.double()).numpy()
    assert np.abs(dX - rx).max() <= 1e-12 * np.abs(rx).max()
    assert np.abs(dW - rw).max() <= 1e-12 * np.abs(rw).max()


def test_backward_delta_cases():
    """A single-tap kernel moves dY back to the tap's offset (data); a single nonzero dY picks
    the input patch under it (filter)."""
    dY = _int_data((1, 1, 4, 5), 24)
    W = np.zeros((1, 1, 3, 3), np.float32)
    W[0, 0, 1, 2] = 1.0
    dX = oracle.conv_bwd_data_fp64(dY, W, 6, 7)
    ref = np.zeros((1, 1, 6, 7))
    ref[0, 0, 1:5, 2:7] = dY[0, 0]
    assert np.array_equal(dX, ref)
    I = _int_data((1, 2, 6, 7), 25)
    d = np.zeros((1, 1, 4, 5), np.float32)
    d[0, 0, 2, 3] = 1.0
    assert np.array_equal(oracle.conv_bwd_filter_fp64(I, d, 3)[0], I[0, :, 2:5, 3:6].astype(np.float64))

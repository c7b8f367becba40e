"""oracle/ -- TEST INFRASTRUCTURE ONLY (the parity oracle).

Plain fp64 CPU direct convolution (Eq. 5, read as "valid"
cross-correlation with W[c'][c][p][q]; see conv_oracle.c's header and DESIGN.md
readings R1-R3).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no
code with ``paper_1809_07851_b200`` (the CUDA product path) and never imports it.

Pins (tests/test_oracle.py): math.fsum brute force on sampled outputs,
hand-computed cases (tests/golden/hand_cases.json), torch fp64 conv2d on CPU,
and the invariants linearity / delta kernel / shift equivariance /
C-additivity / batch independence / channel permutation.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "conv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile conv_oracle.c with gcc (OpenMP, no fast-math).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_conv_fp64.argtypes = [f32p, f32p, f64p] + [ctypes.c_int] * 6
        lib.oracle_conv_fp64.restype = ctypes.c_int
        lib.oracle_conv_fp64_sampled.argtypes = [f32p, f32p, i64p, ctypes.c_longlong, f64p] + [ctypes.c_int] * 6
        lib.oracle_conv_fp64_sampled.restype = ctypes.c_int
        ip = ctypes.POINTER(ctypes.c_int)
        lib.oracle_conv_nd_fp64.argtypes = [f32p, f32p, f64p] + [ctypes.c_int] * 4 + [ip, ip]
        lib.oracle_conv_nd_fp64.restype = ctypes.c_int
        for fn in ("oracle_conv_bwd_data_fp64", "oracle_conv_bwd_filter_fp64"):
            getattr(lib, fn).argtypes = [f32p, f32p, f64p] + [ctypes.c_int] * 6
            getattr(lib, fn).restype = ctypes.c_int
        lib.oracle_num_threads.argtypes = []
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _as_f32(a) -> np.ndarray:
    if hasattr(a, "detach"):  # torch tensor (CPU)
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(a)
    if a.dtype != np.float32:
        raise TypeError("oracle inputs must be float32 (the values the GPU receives)")
    return a


def conv_fp64(I, W) -> np.ndarray:
    """O[b][c'][i][j] = sum_c sum_p sum_q I[b][c][i+p][j+q] * W[c'][c][p][q] in fp64.

    I: [B][C][H][W] float32, W: [C'][C][r][r] float32.  Returns float64
    [B][C'][H-r+1][W-r+1].  PAPER.md P:358-370 (Eq. 5).
    """
    I = _as_f32(I)
    W = _as_f32(W)
    B, C, H, Wd = I.shape
    Co, C2, r, r2 = W.shape
    if C2 != C or r2 != r:
        raise ValueError("shape mismatch between input and weights")
    O = np.empty((B, Co, H - r + 1, Wd - r + 1), dtype=np.float64)
    rc = _load().oracle_conv_fp64(
        I.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        W.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        O.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        B, C, Co, H, Wd, r)
    if rc != 0:
        raise ValueError("oracle_conv_fp64 rejected the shape")
    return O


def conv_fp64_sampled(I, W, idx) -> np.ndarray:
    """The same definition at sampled outputs; idx is an [ns, 4] int array of (b, c', i, j)."""
    I = _as_f32(I)
    W = _as_f32(W)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1, 4))
    B, C, H, Wd = I.shape
    Co, C2, r, _ = W.shape
    if C2 != C:
        raise ValueError("shape mismatch between input and weights")
    out = np.empty(idx.shape[0], dtype=np.float64)
    rc = _load().oracle_conv_fp64_sampled(
        I.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        W.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), idx.shape[0],
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        B, C, Co, H, Wd, r)
    if rc != 0:
        raise ValueError("oracle_conv_fp64_sampled rejected the shape or an index")
    return out


def conv_nd_fp64(I, W) -> np.ndarray:
    """N-dimensional, non-isotropic valid cross-correlation in fp64 (P:926-929 extension of
    Eq. 5): I [B][C][n_0..], W [C'][C][r_0..] float32 with 1..3 spatial axes; returns float64
    [B][C'][n_0 - r_0 + 1 ..]."""
    I = _as_f32(I)
    W = _as_f32(W)
    nd = I.ndim - 2
    if nd < 1 or nd > 3 or W.ndim != I.ndim or W.shape[1] != I.shape[1]:
        raise ValueError("shape mismatch between input and weights")
    B, C = I.shape[:2]
    Co = W.shape[0]
    ins, ks = list(I.shape[2:]), list(W.shape[2:])
    O = np.empty((B, Co) + tuple(a - k + 1 for a, k in zip(ins, ks)), dtype=np.float64)
    ia = (ctypes.c_int * 3)(*ins)
    ka = (ctypes.c_int * 3)(*ks)
    rc = _load().oracle_conv_nd_fp64(
        I.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), W.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        O.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nd, B, C, Co, ia, ka)
    if rc != 0:
        raise ValueError("oracle_conv_nd_fp64 rejected the shape")
    return O


def conv_bwd_data_fp64(dY, W, H: int, Wd: int) -> np.ndarray:
    """dX[b][c][y][x] = sum_{c',p,q} dY[b][c'][y-p][x-q] W[c'][c][p][q] (the adjoint of Eq. 5
    in I) in fp64; dY [B][C'][H-r+1][W-r+1], W [C'][C][r][r] float32 -> [B][C][H][W]."""
    dY, W = _as_f32(dY), _as_f32(W)
    B, Co = dY.shape[:2]
    Co2, C, r, _ = W.shape
    if Co2 != Co or dY.shape[2] != H - r + 1 or dY.shape[3] != Wd - r + 1:
        raise ValueError("shape mismatch")
    dX = np.empty((B, C, H, Wd), dtype=np.float64)
    rc = _load().oracle_conv_bwd_data_fp64(dY.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                           W.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                           dX.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), B, C, Co, H, Wd, r)
    if rc != 0:
        raise ValueError("oracle_conv_bwd_data_fp64 rejected the shape")
    return dX


def conv_bwd_filter_fp64(I, dY, r: int) -> np.ndarray:
    """dW[c'][c][p][q] = sum_{b,i,j} dY[b][c'][i][j] I[b][c][i+p][j+q] (the adjoint of Eq. 5 in W)
    in fp64; I [B][C][H][W], dY [B][C'][H-r+1][W-r+1] float32 -> [C'][C][r][r]."""
    I, dY = _as_f32(I), _as_f32(dY)
    B, C, H, Wd = I.shape
    Co = dY.shape[1]
    if dY.shape[0] != B or dY.shape[2] != H - r + 1 or dY.shape[3] != Wd - r + 1:
        raise ValueError("shape mismatch")
    dW = np.empty((Co, C, r, r), dtype=np.float64)
    rc = _load().oracle_conv_bwd_filter_fp64(I.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                             dY.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                             dW.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), B, C, Co, H, Wd, r)
    if rc != 0:
        raise ValueError("oracle_conv_bwd_filter_fp64 rejected the shape")
    return dW


def num_threads() -> int:
    """OpenMP threads the oracle uses (cpu_baseline.cores)."""
    return int(_load().oracle_num_threads())

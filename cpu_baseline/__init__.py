"""cpu_baseline/ -- the straightforward multithreaded fp32 CPU direct convolution that
bench.py times beside the GPU path (BASELINE.json north_star: "a straightforward
multithreaded CPU direct conv timed on the box's host cores in the same run").
A baseline only: not the parity oracle (oracle/, fp64) and not on the product path."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "direct_fp32.c")
_LIB = os.path.join(_HERE, "libcpudirect.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        # AVX2 + FMA (not -march=native: the .so built here also runs on the GPU box's host CPU)
        cmd = ["gcc", "-O3", "-mavx2", "-mfma", "-fopenmp", "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        f32p = ctypes.POINTER(ctypes.c_float)
        lib.cpu_direct_fp32.argtypes = [f32p, f32p, f32p] + [ctypes.c_int] * 6
        lib.cpu_direct_fp32.restype = ctypes.c_int
        lib.cpu_num_threads.argtypes = []
        lib.cpu_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def conv_fp32(I, W) -> np.ndarray:
    """I [B][C][H][W], W [C'][C][r][r] float32 (numpy or CPU torch) -> float32 output."""
    if hasattr(I, "detach"):
        I = I.detach().cpu().numpy()
    if hasattr(W, "detach"):
        W = W.detach().cpu().numpy()
    I = np.ascontiguousarray(I, dtype=np.float32)
    W = np.ascontiguousarray(W, dtype=np.float32)
    B, C, H, Wd = I.shape
    Co, C2, r, _ = W.shape
    if C2 != C:
        raise ValueError("channel mismatch")
    O = np.empty((B, Co, H - r + 1, Wd - r + 1), dtype=np.float32)
    f32p = ctypes.POINTER(ctypes.c_float)
    st = _load().cpu_direct_fp32(I.ctypes.data_as(f32p), W.ctypes.data_as(f32p), O.ctypes.data_as(f32p),
                                 B, C, Co, H, Wd, r)
    if st != 0:
        raise ValueError("invalid shape")
    return O


def num_threads() -> int:
    return int(_load().cpu_num_threads())

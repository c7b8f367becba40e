"""On-disk cache of full oracle outputs by (config, seed, batch) -- TEST INFRASTRUCTURE.

SURVEY.md sections 5 and 7 (step 1): the fp64 oracle (oracle/, Eq. 5 written out) costs
seconds per full-size BASELINE config, so the full-tensor parity tests compute each
config's output once and keep it as a float64 .npy under ``$FASTCONV_ORACLE_CACHE``
(default ``~/.cache/fastconv_oracle``).  Every cached value is written by this module,
which calls only ``oracle.conv_fp64`` on the seeded ``synth`` inputs; nothing here
touches the CUDA path.  The key carries a digest of the inputs' bytes and of
``oracle/conv_oracle.c``, so a changed generator or oracle never reuses a stale file.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

import oracle
import synth

_ORACLE_SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "conv_oracle.c")


def cache_dir() -> str:
    d = os.environ.get("FASTCONV_ORACLE_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "fastconv_oracle"))
    os.makedirs(d, exist_ok=True)
    return d


def _digest(I, W) -> str:
    h = hashlib.sha256()
    h.update(open(_ORACLE_SRC, "rb").read())
    h.update(np.ascontiguousarray(I.numpy()).tobytes())
    h.update(np.ascontiguousarray(W.numpy()).tobytes())
    return h.hexdigest()[:16]


def full_output(cfg: synth.LayerConfig):
    """(I, W, O): the config's seeded inputs and the oracle's fp64 output (cached on disk)."""
    I, W = synth.make_inputs(cfg)
    key = "%s_seed%d_B%d_%s.npy" % (cfg.name, cfg.seed, cfg.B, _digest(I, W))
    path = os.path.join(cache_dir(), key)
    if os.path.exists(path):
        try:
            O = np.load(path, mmap_mode="r")
            if O.shape == (cfg.B, cfg.Cout, cfg.Ho, cfg.Wo) and O.dtype == np.float64:
                return I, W, O
        except (OSError, ValueError):
            pass
    O = oracle.conv_fp64(I, W)
    try:
        tmp = path + ".%d.tmp" % os.getpid()
        with open(tmp, "wb") as f:
            np.save(f, O)
        os.replace(tmp, path)
    except OSError:
        pass  # a read-only or full cache directory only costs the recomputation
    return I, W, O

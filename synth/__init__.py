"""synth/ -- seeded synthetic workloads shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no transforms, no convolution):
only the layer shapes of BASELINE.json's ``configs`` and the seeded generators
that draw their inputs.  Both ``oracle/`` (via tests) and the CUDA path (via
tests / bench.py) take their inputs from here, so they see identical bits.

Recipe:
  * one ``torch.Generator`` per config, ``manual_seed(seed)``, CPU, fp32;
  * draw order fixed: input I first, then weights W, contiguous NCHW / OIHW;
  * "uniform" = ``torch.rand(...) * 2 - 1`` (U[-1, 1));
  * "normal"  = ``torch.randn(...)`` for I, ``torch.randn(...) * sqrt(2 / (C r^2))``
    (He-normal) for W;
  * multi-GPU ranks slice the globally drawn tensor, they never re-draw.

The paper measured VGG / AlexNet layer *shapes* on CPUs; these
seeded tensors stand in for ImageNet activations and trained weights (none are
available, and timing is data-independent).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

WINOGRAD = "winograd"
REGULAR_FFT = "regular_fft"
GAUSS_FFT = "gauss_fft"
DIRECT = "direct"


@dataclass(frozen=True)
class LayerConfig:
    name: str
    B: int
    C: int
    Cout: int
    H: int
    W: int
    r: int
    seed: int
    dist: str  # "uniform" or "normal"
    # (method, m) pairs exercised for this config (BASELINE.json configs)
    runs: tuple = field(default_factory=tuple)

    @property
    def Ho(self) -> int:
        return self.H - self.r + 1

    @property
    def Wo(self) -> int:
        return self.W - self.r + 1

    @property
    def direct_flops(self) -> float:
        """2*B*C*C'*Ho*Wo*r^2: the direct-convolution FLOPs (BASELINE.json metric)."""
        return 2.0 * self.B * self.C * self.Cout * self.Ho * self.Wo * self.r * self.r

    def with_batch(self, B: int) -> "LayerConfig":
        return LayerConfig(self.name, B, self.C, self.Cout, self.H, self.W, self.r,
                           self.seed, self.dist, self.runs)


def _fft(ms):
    return tuple((m_, k) for k in ms for m_ in (REGULAR_FFT, GAUSS_FFT))


# BASELINE.json configs[0..4]
CONFIGS = {
    "tiny": LayerConfig("tiny", 1, 4, 4, 16, 16, 3, 1, "uniform",
                        ((REGULAR_FFT, 6), (GAUSS_FFT, 6), (WINOGRAD, 2), (WINOGRAD, 4))),
    "vgg3_2": LayerConfig("vgg3_2", 64, 256, 256, 58, 58, 3, 2, "normal",
                          ((WINOGRAD, 2), (WINOGRAD, 4), (WINOGRAD, 6)) + _fft((8, 14, 22, 30))),
    "vgg1_2": LayerConfig("vgg1_2", 64, 64, 64, 226, 226, 3, 3, "normal",
                          ((WINOGRAD, 2), (WINOGRAD, 4), (WINOGRAD, 6)) + _fft((14, 25, 30))),
    "k5": LayerConfig("k5", 128, 96, 256, 31, 31, 5, 4, "normal",
                      ((WINOGRAD, 2),) + _fft((9, 14, 27))),
    "deep": LayerConfig("deep", 64, 512, 512, 16, 16, 3, 5, "normal",
                        ((WINOGRAD, 2), (WINOGRAD, 4), (WINOGRAD, 6)) + _fft((7, 14))),
}


def make_inputs(cfg: LayerConfig, seed: int | None = None):
    """Draw (I, W) for ``cfg`` on the CPU as contiguous fp32 torch tensors."""
    g = torch.Generator().manual_seed(cfg.seed if seed is None else seed)
    ishape = (cfg.B, cfg.C, cfg.H, cfg.W)
    wshape = (cfg.Cout, cfg.C, cfg.r, cfg.r)
    if cfg.dist == "uniform":
        I = torch.rand(ishape, generator=g, dtype=torch.float32) * 2 - 1
        W = torch.rand(wshape, generator=g, dtype=torch.float32) * 2 - 1
    elif cfg.dist == "normal":
        I = torch.randn(ishape, generator=g, dtype=torch.float32)
        W = torch.randn(wshape, generator=g, dtype=torch.float32) * math.sqrt(2.0 / (cfg.C * cfg.r * cfg.r))
    else:
        raise ValueError(cfg.dist)
    return I.contiguous(), W.contiguous()


def custom(B, C, Cout, H, W, r, seed=0, dist="uniform", name="custom") -> LayerConfig:
    return LayerConfig(name, B, C, Cout, H, W, r, seed, dist, ())


def sample_output_indices(cfg: LayerConfig, n: int, seed: int = 1234) -> np.ndarray:
    """[n + 4*B', 4] int64 (b, c', i, j): n uniform samples plus the 4 spatial corners
    of the first and last (b, c') planes (where ragged tiles and borders live)."""
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, cfg.B, n), rng.integers(0, cfg.Cout, n),
                    rng.integers(0, cfg.Ho, n), rng.integers(0, cfg.Wo, n)], axis=1)
    corners = []
    for b, co in ((0, 0), (cfg.B - 1, cfg.Cout - 1)):
        for i in (0, cfg.Ho - 1):
            for j in (0, cfg.Wo - 1):
                corners.append((b, co, i, j))
    return np.concatenate([idx, np.asarray(corners, dtype=np.int64)], axis=0).astype(np.int64)


"""Sampling configuration and the warp / sample primitives on the GPU.

API of the reference `speckit.sampling` (pkg/src/speckit/sampling.py): the
dataclass and its validation are host logic; `apply_warp` and `sample` run the
canonical float64 row kernels (csrc/warp_rows.cuh) -- temperature 0 is a
one-hot argmax with the lowest id winning ties, T != 1 rescales and
renormalises, top-p keeps the smallest (prob desc, id asc) prefix whose
cumulative mass reaches top_p - 1e-9, and `sample` consumes exactly one uniform
and inverts the CDF over ascending ids.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import CounterRng

DIST_ATOL = 1e-9


@dataclass(frozen=True)
class SamplingConfig:
    """sampling.py:21-41"""

    temperature: float = 1.0
    top_p: float = 1.0
    seed: int = 0
    max_new_tokens: int = 16

    def __post_init__(self) -> None:
        if self.temperature < 0:
            raise ValueError(f"temperature must be >= 0, got {self.temperature}")
        if not 0 < self.top_p <= 1:
            raise ValueError(f"top_p must be in (0, 1], got {self.top_p}")
        if self.max_new_tokens < 0:
            raise ValueError(f"max_new_tokens must be >= 0, got {self.max_new_tokens}")

    @property
    def is_identity(self) -> bool:
        return self.temperature == 1.0 and self.top_p >= 1.0


def validate_distribution(probs: np.ndarray) -> np.ndarray:
    """sampling.py:44-56 (host-side argument check)."""
    p = np.asarray(probs, dtype=np.float64)
    if p.ndim != 1:
        raise ValueError(f"distribution must be 1-D, got shape {p.shape}")
    if p.size == 0:
        raise ValueError("distribution must be non-empty")
    if np.any(p < 0):
        raise ValueError("distribution has negative entries")
    total = float(p.sum())
    if abs(total - 1.0) > DIST_ATOL:
        raise ValueError(f"distribution sums to {total!r}, expected 1 within {DIST_ATOL}")
    return p


def _device_rows(dist):
    import torch

    if isinstance(dist, torch.Tensor):
        t = dist
    else:
        t = torch.as_tensor(np.asarray(dist, dtype=np.float64))
    if not t.is_cuda:
        t = t.cuda()
    return t


def apply_warp(dist, cfg: SamplingConfig) -> np.ndarray:
    """Temperature-scale then nucleus-truncate one distribution on the GPU.

    Accepts a float64 probability row (numpy or CUDA tensor) or an fp32 logits
    CUDA tensor; returns the warped float64 row as numpy.
    """
    import torch

    from . import kernels as K

    t = _device_rows(dist)
    if cfg.is_identity and t.dtype == torch.float64:
        return t.double().cpu().numpy()
    out = K.warp_rows(t.reshape(1, -1), cfg.temperature, cfg.top_p)
    return out[0].cpu().numpy()


def sample(dist, rng: CounterRng) -> int:
    """Inverse-CDF sample over ascending ids, consuming exactly one draw."""
    from . import kernels as K

    t = _device_rows(dist).double().reshape(1, -1)
    u = rng.uniform()
    return int(K.sample_rows(t, np.array([u]))[0])

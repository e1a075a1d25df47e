"""Load-balancing statistics (sb/metrics.py:59-86) for GPU load maps.

The render epilogue already reduces the load map to exact integer moments
(sum, sum of squares, min, max); ``load_loss`` turns them into the population
standard deviation with exact rational arithmetic, so it agrees with the
reference's two-pass numpy value to ~1 ulp (the reference test bound is 1e-9
relative, sb tests/test_acceptance.py:157-166).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

PSNR_IDENTICAL_SENTINEL = 999.0


def _moments(load_map):
    """(n, sum, sum_sq, min, max) of a LoadMap (CUDA tensor or numpy)."""
    counts = load_map.counts if hasattr(load_map, "counts") else load_map
    try:
        import torch

        if isinstance(counts, torch.Tensor):
            c = counts.reshape(-1).to(torch.int64)
            n = c.numel()
            if n == 0:
                raise ValueError("load map is empty")
            return (n, int(c.sum().item()), int((c * c).sum().item()), int(c.min().item()),
                    int(c.max().item()))
    except ImportError:  # pragma: no cover
        pass
    c = np.asarray(counts, dtype=np.int64).ravel()
    if c.size == 0:
        raise ValueError("load map is empty")
    return c.size, int(c.sum()), int((c * c).sum()), int(c.min()), int(c.max())


def std_from_moments(n: int, s: int, s2: int) -> float:
    """Population std from exact integer moments: sqrt((n*S2 - S1^2) / n^2)."""
    var = Fraction(n * s2 - s * s, n * n)
    return math.sqrt(var) if var > 0 else 0.0


def load_loss(load_map) -> float:
    """Population standard deviation of the per-pixel composited counts (sb/metrics.py:80-86)."""
    n, s, s2, _, _ = _moments(load_map)
    return std_from_moments(n, s, s2)


@dataclass(frozen=True)
class LoadStats:
    """Summary of a load map (sb/metrics.py:59-77)."""

    mean: float
    std: float
    min: int
    max: int
    histogram: np.ndarray

    @classmethod
    def from_load_map(cls, load_map) -> "LoadStats":
        n, s, s2, mn, mx = _moments(load_map)
        counts = load_map.counts if hasattr(load_map, "counts") else load_map
        try:
            import torch

            if isinstance(counts, torch.Tensor):
                hist = torch.bincount(counts.reshape(-1).to(torch.int64)).cpu().numpy()
            else:
                hist = np.bincount(np.asarray(counts).ravel())
        except ImportError:  # pragma: no cover
            hist = np.bincount(np.asarray(counts).ravel())
        return cls(mean=s / n, std=std_from_moments(n, s, s2), min=mn, max=mx, histogram=hist)

    @classmethod
    def from_moments(cls, n: int, s: int, s2: int, mn: int, mx: int, histogram=None) -> "LoadStats":
        """From the render epilogue's exact moments (no extra pass over the map)."""
        return cls(mean=s / n, std=std_from_moments(n, s, s2), min=mn, max=mx,
                   histogram=np.asarray(histogram if histogram is not None else [], dtype=np.int64))


def psnr(a, b) -> float:
    """PSNR in dB of unit-range images; inf when identical (sb/metrics.py:100-106)."""
    pa = a.pixels if hasattr(a, "pixels") else a
    pb = b.pixels if hasattr(b, "pixels") else b
    pa = pa.cpu().numpy() if hasattr(pa, "cpu") else np.asarray(pa)
    pb = pb.cpu().numpy() if hasattr(pb, "cpu") else np.asarray(pb)
    if pa.shape != pb.shape:
        raise ValueError("image dimensions differ")
    mse = float(np.mean((pa.astype(np.float64) - pb.astype(np.float64)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)

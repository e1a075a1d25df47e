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


# ---------------------------------------------------------------------------
# Image terms and the load-balancing objective (sb/metrics.py:39-143), on the
# GPU (csrc/adr_metrics.cu), plus the toy optimizer (sb/metrics.py:167-216)
# as a batched GPU loop — SURVEY.md §8f row 1.
# ---------------------------------------------------------------------------

_SSIM_WINDOW = 11
_SSIM_SIGMA = 1.5
_SSIM_C1 = 0.01 ** 2
_SSIM_C2 = 0.03 ** 2


@dataclass(frozen=True)
class LossWeights:
    """Non-negative weights for (L1, SSIM, load) summing to one (sb/metrics.py:39-53)."""

    lambda_l1: float = 0.44
    lambda_ssim: float = 0.11
    lambda_load: float = 0.45

    def __post_init__(self) -> None:
        for name in ("lambda_l1", "lambda_ssim", "lambda_load"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")
        total = self.lambda_l1 + self.lambda_ssim + self.lambda_load
        if abs(total - 1.0) > 1e-9:
            raise ValueError(f"weights must sum to 1 (got {total!r})")


DEFAULT_WEIGHTS = LossWeights()


def _ssim_window() -> np.ndarray:
    """sb/metrics.py:108-111, the same numpy expression (host)."""
    offsets = np.arange(_SSIM_WINDOW, dtype=np.float64) - _SSIM_WINDOW // 2
    w = np.exp(-(offsets ** 2) / (2.0 * _SSIM_SIGMA ** 2))
    return w / w.sum()


_WINDOW = None


def _window_ptr():
    import ctypes

    global _WINDOW
    if _WINDOW is None:
        _WINDOW = (ctypes.c_double * 11)(*_ssim_window().tolist())
    return _WINDOW


def _device_pixels(img, device):
    import torch

    p = img.pixels if hasattr(img, "pixels") else img
    t = p if isinstance(p, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32))
    return t.to(device=device, dtype=torch.float32).contiguous()


class ImageLoss:
    """Asynchronous (L1, SSIM) of (H, W, 3) float32 CUDA images into a
    float64 device slot; reusable scratch for one image size."""

    def __init__(self, width: int, height: int, device):
        import torch

        from . import _lib

        self.width, self.height, self.device = int(width), int(height), torch.device(device)
        n = _lib.lib().adr_image_loss_scratch_bytes(self.width, self.height)
        self.scratch = torch.empty(max(int(n), 8), dtype=torch.uint8, device=self.device)

    def __call__(self, a, b, out, stream=None) -> None:
        import torch

        from . import _lib

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(_lib.lib().adr_image_losses(
            _lib.ptr(a), _lib.ptr(b), self.width, self.height, _window_ptr(), _SSIM_C1, _SSIM_C2,
            _lib.ptr(out), _lib.ptr(self.scratch), self.scratch.numel(), _lib.stream_handle(st)))


def _check_dims(a, b) -> None:
    if (a.width, a.height) != (b.width, b.height):
        raise ValueError("image dimensions differ")


def _image_terms(a, b):
    import torch

    _check_dims(a, b)
    dev = torch.device("cuda")
    pa, pb = _device_pixels(a, dev), _device_pixels(b, dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    ImageLoss(a.width, a.height, dev)(pa, pb, out)
    l1, s = out.tolist()
    return l1, s


def l1_loss(a, b) -> float:
    """Mean absolute per-channel difference (sb/metrics.py:94-97), fp64 on the GPU."""
    return _image_terms(a, b)[0]


def ssim(a, b) -> float:
    """Mean SSIM, 11x11 Gaussian window sigma 1.5, zero padding
    (sb/metrics.py:120-140), fp64 on the GPU."""
    return _image_terms(a, b)[1]


def _combine(weights: LossWeights, l1: float, s: float, load: float) -> float:
    """total_loss's accumulation order (sb/metrics.py:143-152)."""
    value = 0.0
    if weights.lambda_l1:
        value += weights.lambda_l1 * l1
    if weights.lambda_ssim:
        value += weights.lambda_ssim * (1.0 - s)
    if weights.lambda_load:
        value += weights.lambda_load * load
    return value


def total_loss(rendered, reference, load_map, weights: LossWeights = DEFAULT_WEIGHTS) -> float:
    """Weighted L1 + (1 - SSIM) + load-balancing loss (sb/metrics.py:143-152)."""
    l1, s = _image_terms(rendered, reference)
    return _combine(weights, l1, s, load_loss(load_map) if weights.lambda_load else 0.0)


@dataclass(eq=False)
class BalanceStepResult:
    scene: object
    loss_before: float
    loss_after: float


def replace_opacity(g, value: float):
    """sb/metrics.py:213-216."""
    from .scene import Gaussian3D

    return Gaussian3D(center=g.center.copy(), scale=g.scale.copy(), rotation=g.rotation.copy(),
                      opacity=value, sh_coeffs=g.sh_coeffs.copy())


def toy_balance_step(scene, cam, reference, weights: LossWeights, step: float, alpha_low: float = None,
                     fd_epsilon: float = 0.02, mode=None, threads: int = 1) -> BalanceStepResult:
    """One central-finite-difference descent step on the opacities
    (sb/metrics.py:167-210), with every probe rendered on the GPU.

    The 2N + 1 evaluations (base + a hi/lo probe per Gaussian) are independent
    frames of the same scene that differ in one opacity: they are enqueued
    back to back on one stream through one persistent Rasterizer, each
    followed by the fp64 L1/SSIM kernel into its own slot and a copy of the
    epilogue's exact load moments, with a single host synchronisation for the
    whole batch.  Then the step and one more frame for ``loss_after``.
    ``threads`` is accepted for signature compatibility.
    """
    import torch

    from .pipeline import Rasterizer
    from .projection import ALPHA_LOW, CullingMode
    from .scene import DeviceScene, Scene

    alpha_low = ALPHA_LOW if alpha_low is None else alpha_low
    mode = CullingMode.AABB if mode is None else CullingMode(mode)
    if step <= 0:
        raise ValueError("step must be positive")
    if len(scene) > 500:
        raise ValueError("toy optimizer is limited to 500 Gaussians")
    if scene.sh_degree != 0:
        raise ValueError("toy optimizer requires SH degree 0")
    dev = torch.device("cuda")
    arrays = scene.as_arrays()
    n = len(arrays.opacities)
    base = np.asarray(arrays.opacities, dtype=np.float64)
    hi = np.array([min(o + fd_epsilon, 1.0) for o in base.tolist()])
    lo = np.array([max(o - fd_epsilon, 1e-4) for o in base.tolist()])
    ref = _device_pixels(reference, dev)
    ds = DeviceScene.from_arrays(arrays, 0, dev, torch.float64)
    rast = Rasterizer(cam.width, cam.height, n, device=dev, timing=False)
    loss_k = ImageLoss(cam.width, cam.height, dev)

    def run(opmat: np.ndarray):
        """Loss of every opacity row (fp64) — all frames async, one sync."""
        ops = torch.from_numpy(opmat).to(dev)
        v = ops.shape[0]
        while True:
            terms = torch.empty((v, 2), dtype=torch.float64, device=dev)
            moments = torch.empty((v, 3), dtype=torch.int64, device=dev)
            pairs = torch.empty(v, dtype=torch.int64, device=dev)
            for k in range(v):
                dk = DeviceScene(ds.centers, ds.scales, ds.rotations, ops[k], ds.sh, 0)
                rast.launch(dk, cam, mode, alpha_low)
                loss_k(rast.pixels, ref, terms[k])
                moments[k].copy_(rast.stats, non_blocking=True)
                pairs[k].copy_(rast.counters[0], non_blocking=True)
            torch.cuda.synchronize(dev)
            pmax = int(pairs.max().item()) if v else 0
            if pmax <= rast.cap:
                break
            rast.fit_capacity(int(pmax * 1.25) + 1024)
        t = terms.cpu().tolist()
        mo = moments.cpu().tolist()
        npx = cam.width * cam.height
        out = []
        for k in range(v):
            load = std_from_moments(npx, int(mo[k][0]), int(mo[k][1])) if weights.lambda_load else 0.0
            out.append(_combine(weights, t[k][0], t[k][1], load))
        return out

    rows = [base]
    for i in range(n):
        if hi[i] <= lo[i]:
            continue
        rows.append(np.where(np.arange(n) == i, hi[i], base))
        rows.append(np.where(np.arange(n) == i, lo[i], base))
    losses = run(np.stack(rows))
    loss_before = losses[0]
    grad = np.zeros(n)
    j = 1
    for i in range(n):
        if hi[i] <= lo[i]:
            continue
        grad[i] = (losses[j] - losses[j + 1]) / (hi[i] - lo[i])
        j += 2
    new_op = np.array([float(np.clip(base[i] - step * grad[i], 1e-4, 1.0)) for i in range(n)])
    loss_after = run(new_op[None, :])[0]
    if isinstance(scene, Scene) or hasattr(scene, "gaussians"):
        new_scene = Scene(gaussians=[replace_opacity(g, float(new_op[i])) for i, g in enumerate(scene.gaussians)],
                          sh_degree=scene.sh_degree)
    else:
        new_scene = arrays._replace(opacities=new_op)
    return BalanceStepResult(scene=new_scene, loss_before=loss_before, loss_after=loss_after)

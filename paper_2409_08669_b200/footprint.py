"""Per-Gaussian footprint mathematics on the host (fp64), the scalar side of
the reference's public surface (sb/projection.py:52-289, :423-441;
sb/render.py:57-125).

These are the closed forms of the paper's culling (§4.2 adaptive radius,
§4.3 axis-aligned bounding box) for ONE Gaussian, used by tests, tooling and
anyone reasoning about a single splat: the bulk path computes the same
quantities in ``csrc/adr_preprocess.cu`` for millions of Gaussians at once.
``project_gaussian`` runs that GPU preprocess on a one-Gaussian scene, like
the reference runs its batched preprocess (sb/projection.py:427-428).
``composite_pixels`` is the host blend used with a ``present_fn`` mask (the
reference's brute-force renderer interface); the GPU path never calls it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .projection import ALPHA_LOW, BASE_RADIUS_MULTIPLIER, COV_DILATION, CullingMode

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
         0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


@dataclass(frozen=True)
class CullExtent:
    """Footprint half-widths in pixels (sb/projection.py:52-58)."""

    mode: CullingMode
    rx: int
    ry: int


@dataclass(frozen=True)
class EllipseCoefficients:
    """Iso-opacity boundary a x^2 + b y^2 + c x y + d = 0 (sb/projection.py:61-68)."""

    a: float
    b: float
    c: float
    d: float


@dataclass(frozen=True, eq=False)
class ProjectedGaussian:
    """One screen-space splat (sb/projection.py:71-83)."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    lambda_max: float
    extent: CullExtent


def _sh_terms(x, y, z, degree: int):
    """Real SH basis values (with the reference's signs and constants) in the
    order the coefficients are stored, as scalar or array expressions."""
    terms = [SH_C0]
    if degree > 0:
        terms += [-SH_C1 * y, SH_C1 * z, -SH_C1 * x]
    if degree > 1:
        xx, yy, zz = x * x, y * y, z * z
        terms += [SH_C2[0] * (x * y), SH_C2[1] * (y * z), SH_C2[2] * (2.0 * zz - xx - yy),
                  SH_C2[3] * (x * z), SH_C2[4] * (xx - yy)]
        if degree > 2:
            terms += [SH_C3[0] * y * (3.0 * xx - yy), SH_C3[1] * (x * y) * z,
                      SH_C3[2] * y * (4.0 * zz - xx - yy), SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                      SH_C3[4] * x * (4.0 * zz - xx - yy), SH_C3[5] * z * (xx - yy),
                      SH_C3[6] * x * (xx - 3.0 * yy)]
    return terms


def evaluate_sh(coeffs, direction, degree: int) -> np.ndarray:
    """RGB of one Gaussian seen along unit ``direction``: SH degree 0..3, +0.5,
    clipped to [0, 1] on both sides (sb/projection.py:128-163)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    k = (degree + 1) ** 2
    if coeffs.shape != (k, 3):
        raise ValueError(f"expected {k} coefficient triples for degree {degree}, got {coeffs.shape}")
    x, y, z = (float(v) for v in np.asarray(direction, dtype=np.float64).reshape(3))
    out = np.zeros(3)
    for basis, c in zip(_sh_terms(x, y, z, degree), coeffs):
        out = out + basis * c
    return np.clip(out + 0.5, 0.0, 1.0)


def quaternion_to_rotation(q) -> np.ndarray:
    """Unit quaternion(s) (..., 4) wxyz -> rotation matrices (..., 3, 3)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = (q[..., i] for i in range(4))
    return np.stack([
        np.stack([1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)], -1),
        np.stack([2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)], -1),
        np.stack([2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)], -1),
    ], -2)


def build_covariance3d(scale, rotation) -> np.ndarray:
    """Sigma = (R S)(R S)^T from per-axis scales and a unit quaternion
    (sb/projection.py:187-197)."""
    s = np.asarray(scale, dtype=np.float64).reshape(3)
    q = np.asarray(rotation, dtype=np.float64).reshape(4)
    if not (np.isfinite(s).all() and np.isfinite(q).all()):
        raise ValueError("scale and rotation must be finite")
    if (s <= 0).any():
        raise ValueError("scale components must be positive")
    rs = quaternion_to_rotation(q) * s
    return rs @ rs.T


def _pd(cov2d):
    c = np.asarray(cov2d, dtype=np.float64)
    sxx, syy, sxy = float(c[0, 0]), float(c[1, 1]), float(c[0, 1])
    det = sxx * syy - sxy * sxy
    if sxx <= 0 or det <= 0:
        raise ValueError("covariance must be positive definite")
    return sxx, syy, sxy, det


def eigen_extents(cov2d) -> tuple:
    """(lambda_max, lambda_min) of a positive-definite 2x2 (sb/projection.py:200-209)."""
    sxx, syy, _, det = _pd(cov2d)
    mid = 0.5 * (sxx + syy)
    disc = math.sqrt(max(mid * mid - det, 0.0))
    return mid + disc, mid - disc


def radius_baseline(lambda_max: float) -> int:
    """ceil(3 sqrt(lambda_max)), the 3-sigma square (sb/projection.py:212-216)."""
    if lambda_max <= 0:
        raise ValueError("lambda_max must be positive")
    return math.ceil(BASE_RADIUS_MULTIPLIER * math.sqrt(lambda_max))


def bounding_circle_radius(lambda_max: float, sigma: float, alpha_low: float) -> float:
    """sqrt(2 lambda_max ln(sigma / alpha_low)): the circle bounding the ellipse
    where sigma * exp(-d^2 / 2) >= alpha_low (paper §4.2; sb/projection.py:219-225)."""
    return math.sqrt(2.0 * lambda_max * math.log(sigma / alpha_low))


def radius_adaptive(lambda_max: float, sigma: float, alpha_low: float):
    """Adaptive radius: ceil(min(circle, 3 sqrt(lambda_max))), None when culled
    (sigma <= alpha_low or radius < 1; sb/projection.py:228-243)."""
    if lambda_max <= 0:
        raise ValueError("lambda_max must be positive")
    if not 0.0 < alpha_low < 1.0:
        raise ValueError("alpha_low must lie in (0, 1)")
    if sigma <= alpha_low:
        return None
    r = math.ceil(min(bounding_circle_radius(lambda_max, sigma, alpha_low),
                      BASE_RADIUS_MULTIPLIER * math.sqrt(lambda_max)))
    return r if r >= 1 else None


def ellipse_coefficients(cov2d, sigma: float, alpha_low: float) -> EllipseCoefficients:
    """Iso-opacity boundary of one splat (sb/projection.py:246-262):
    syy x^2 + sxx y^2 - 2 sxy x y - 2 det ln(sigma / alpha_low) <= 0."""
    if sigma <= alpha_low:
        raise ValueError("sigma must exceed alpha_low (the caller culls first)")
    sxx, syy, sxy, det = _pd(cov2d)
    return EllipseCoefficients(a=syy, b=sxx, c=-2.0 * sxy, d=-2.0 * det * math.log(sigma / alpha_low))


def bounding_box_halfwidths(cov2d, sigma: float, alpha_low: float) -> tuple:
    """Per-axis half-widths sqrt(2 s_xx ln(sigma/alpha_low)), sqrt(2 s_yy ...)
    of the iso-opacity ellipse (paper §4.3; sb/projection.py:265-270)."""
    c = np.asarray(cov2d, dtype=np.float64)
    lr = math.log(sigma / alpha_low)
    return math.sqrt(2.0 * float(c[0, 0]) * lr), math.sqrt(2.0 * float(c[1, 1]) * lr)


def aabb_extents(cov2d, sigma: float, alpha_low: float, lambda_max: float):
    """(rx, ry) per-axis footprint, each clamped by the 3-sigma radius, or None
    when culled (sb/projection.py:273-286)."""
    if not 0.0 < alpha_low < 1.0:
        raise ValueError("alpha_low must lie in (0, 1)")
    if sigma <= alpha_low:
        return None
    hx, hy = bounding_box_halfwidths(cov2d, sigma, alpha_low)
    r_o = BASE_RADIUS_MULTIPLIER * math.sqrt(lambda_max)
    rx, ry = math.ceil(min(hx, r_o)), math.ceil(min(hy, r_o))
    if rx < 1 or ry < 1:
        return None
    return rx, ry


def project_gaussian(g, cam, alpha_low: float = ALPHA_LOW, mode: CullingMode = CullingMode.AABB,
                     dilation: float = COV_DILATION):
    """One Gaussian through the GPU preprocess; None when culled
    (sb/projection.py:423-441)."""
    from .projection import preprocess
    from .scene import Scene

    deg = int(round(math.sqrt(len(g.sh_coeffs)))) - 1
    proj = preprocess(Scene(gaussians=[g], sh_degree=deg), cam, mode=mode, alpha_low=alpha_low,
                      dilation=dilation).to_numpy()
    if not proj["valid"][0]:
        return None
    sxx, syy, sxy = (float(v) for v in proj["cov2d"][0])
    mode = CullingMode(mode)
    return ProjectedGaussian(mean2d=proj["mean2d"][0].astype(np.float64),
                             cov2d=np.array([[sxx, sxy], [sxy, syy]]),
                             conic=proj["conic"][0].astype(np.float64), depth=float(proj["depth"][0]),
                             color=proj["color"][0].astype(np.float64), opacity=float(proj["opacity"][0]),
                             lambda_max=float(proj["lambda_max"][0]),
                             extent=CullExtent(mode=mode, rx=int(proj["ext_x"][0]), ry=int(proj["ext_y"][0])))


def composite_pixels(px, py, order, proj, alpha_low: float, background, term_threshold: float = 1e-4,
                     present_fn=None):
    """Front-to-back blend of the pair sequence ``order`` over a flat block of
    pixels on the host (sb/render.py:57-125): fp32 throughout, numpy's float32
    exp, alpha clamp 0.99, skip below alpha_low, stop after the contribution
    that takes T below the threshold.  ``present_fn(idx)`` masks pairs per
    pixel; absent pairs are exact no-ops.  Returns (rgb (n,3) float32 clamped
    to [0,1], counts (n,) int32)."""
    p = proj.to_numpy() if hasattr(proj, "to_numpy") else proj
    px = np.asarray(px, dtype=np.float32)
    py = np.asarray(py, dtype=np.float32)
    order = np.asarray(order, dtype=np.int64)
    n = len(px)
    f32 = np.float32
    a_low, term, clamp = f32(alpha_low), f32(term_threshold), f32(0.99)
    T = np.ones(n, dtype=np.float32)
    C = np.zeros((n, 3), dtype=np.float32)
    cnt = np.zeros(n, dtype=np.int32)
    live = np.ones(n, dtype=bool)
    mean = np.asarray(p["mean2d"] if isinstance(p, dict) else p.mean2d, dtype=np.float32)
    con = np.asarray(p["conic"] if isinstance(p, dict) else p.conic, dtype=np.float32)
    op = np.asarray(p["opacity"] if isinstance(p, dict) else p.opacity, dtype=np.float32)
    col = np.asarray(p["color"] if isinstance(p, dict) else p.color, dtype=np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        for chunk in range(0, len(order), 2048):
            idx = order[chunk:chunk + 2048]
            mask = present_fn(idx) if present_fn is not None else None
            for k, g in enumerate(idx):
                if not live.any():
                    break
                dx = px - mean[g, 0]
                dy = py - mean[g, 1]
                power = f32(-0.5) * (con[g, 0] * dx * dx + con[g, 2] * dy * dy) - con[g, 1] * dx * dy
                alpha = np.minimum(op[g] * np.exp(power), clamp)
                on = live & (alpha >= a_low)
                if mask is not None:
                    on &= mask[k]
                w = np.where(on, alpha * T, f32(0))
                C = (C + w[:, None] * col[g][None, :]).astype(np.float32)
                T = np.where(on, T * (f32(1) - alpha), T)
                cnt += on
                live &= ~(on & (T < term))
    rgb = C + T[:, None] * np.asarray(background, dtype=np.float32)[None, :]
    return np.clip(rgb, 0.0, 1.0).astype(np.float32), cnt

"""Scene model on the input side of the boundary (sb/scene.py).

``Camera``, ``Gaussian3D``, ``Scene``, ``SceneArrays``, ``SyntheticSpec`` and
``generate_synthetic`` keep the reference's fields, validation and random
draws, so reference scenes and ours are interchangeable inputs.  On top of
that, ``DeviceScene`` holds the SoA arrays as CUDA tensors (fp32 or fp64) —
the form the kernels consume — so large scenes never pass through Python
objects (``Scene.as_arrays`` costs seconds per million Gaussians).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .errors import SceneValidationError

SH_C0 = 0.28209479177387814
MAX_SH_DEGREE = 3
_ROTATION_ORTHO_TOL = 1e-5


@dataclass(eq=False)
class Gaussian3D:
    """One anisotropic Gaussian (sb/scene.py:43-71): center, per-axis scale,
    unit quaternion (w, x, y, z), opacity, SH coefficients ((deg+1)^2, 3)."""

    center: np.ndarray
    scale: np.ndarray
    rotation: np.ndarray
    opacity: float
    sh_coeffs: np.ndarray

    def __post_init__(self) -> None:
        self.center = np.asarray(self.center, dtype=np.float64).reshape(3)
        self.scale = np.asarray(self.scale, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.opacity = float(self.opacity)
        self.sh_coeffs = np.asarray(self.sh_coeffs, dtype=np.float64).reshape(-1, 3)


class SceneArrays(NamedTuple):
    """Dense fp64 per-Gaussian arrays (sb/scene.py:105-110)."""

    centers: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray


@dataclass(eq=False)
class Scene:
    """Ordered Gaussians with a common SH degree (sb/scene.py:75-102)."""

    gaussians: list
    sh_degree: int = 0

    def __len__(self) -> int:
        return len(self.gaussians)

    def as_arrays(self) -> SceneArrays:
        k = (self.sh_degree + 1) ** 2
        if not self.gaussians:
            return SceneArrays(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)),
                               np.zeros(0), np.zeros((0, k, 3)))
        return SceneArrays(
            centers=np.stack([g.center for g in self.gaussians]),
            scales=np.stack([g.scale for g in self.gaussians]),
            rotations=np.stack([g.rotation for g in self.gaussians]),
            opacities=np.array([g.opacity for g in self.gaussians]),
            sh=np.stack([g.sh_coeffs for g in self.gaussians]),
        )


@dataclass(frozen=True, eq=False)
class Camera:
    """Pinhole camera with a world-to-camera 4x4 transform (sb/scene.py:114-200).

    A view-space point (x, y, z) projects to pixel
    (fx*x/z + (W-1)/2, fy*y/z + (H-1)/2): pixel centres are integers.
    """

    view_matrix: np.ndarray
    fx: float
    fy: float
    width: int
    height: int
    near_plane: float = 0.2
    background: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self) -> None:
        vm = np.asarray(self.view_matrix, dtype=np.float64).reshape(4, 4)
        object.__setattr__(self, "view_matrix", vm)
        rot = vm[:3, :3]
        if not np.allclose(rot @ rot.T, np.eye(3), atol=_ROTATION_ORTHO_TOL):
            raise ValueError("view_matrix rotation block is not orthonormal")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.near_plane <= 0:
            raise ValueError("near_plane must be positive")
        bg = tuple(float(c) for c in self.background)
        if len(bg) != 3 or any(not 0.0 <= c <= 1.0 for c in bg):
            raise ValueError("background must be an RGB triple in [0, 1]")
        object.__setattr__(self, "background", bg)

    @property
    def rotation(self) -> np.ndarray:
        return self.view_matrix[:3, :3]

    @property
    def translation(self) -> np.ndarray:
        return self.view_matrix[:3, 3]

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @classmethod
    def from_lookat(cls, position, target, up=(0.0, 1.0, 0.0), fov_y_deg: float = 60.0,
                    width: int = 256, height: int = 256, near_plane: float = 0.2,
                    background=(0.0, 0.0, 0.0)) -> "Camera":
        position = np.asarray(position, dtype=np.float64).reshape(3)
        target = np.asarray(target, dtype=np.float64).reshape(3)
        up = np.asarray(up, dtype=np.float64).reshape(3)
        fwd = target - position
        n = np.linalg.norm(fwd)
        if n < 1e-12:
            raise ValueError("camera position and target coincide")
        z_axis = fwd / n
        x_axis = np.cross(up, z_axis)
        n = np.linalg.norm(x_axis)
        if n < 1e-12:
            raise ValueError("up vector is parallel to the view direction")
        x_axis /= n
        y_axis = np.cross(z_axis, x_axis)
        rot = np.stack([x_axis, y_axis, z_axis])
        vm = np.eye(4)
        vm[:3, :3] = rot
        vm[:3, 3] = -rot @ position
        f = 0.5 * height / math.tan(math.radians(fov_y_deg) / 2.0)
        return cls(view_matrix=vm, fx=f, fy=f, width=int(width), height=int(height),
                   near_plane=near_plane, background=background)


@dataclass(frozen=True)
class SyntheticSpec:
    """Distribution parameters of the seeded generator (sb/scene.py:204-210)."""

    extent: float = 1.0
    scale_range: tuple = (0.02, 0.08)
    anisotropy_range: tuple = (1.0, 4.0)
    opacity_range: tuple = (0.05, 0.95)


def synthetic_arrays(seed: int, count: int, spec: SyntheticSpec | None = None,
                     sh_degree: int = 0, sh_rest_sigma: float = 0.3,
                     float32: bool = False) -> SceneArrays:
    """Vectorised seeded scene: the same draws, in the same order, as
    ``generate_synthetic`` (sb/scene.py:241-259), plus optional higher-order SH
    coefficients N(0, sh_rest_sigma^2) drawn afterwards from the same stream.

    ``float32=True`` rounds every value to fp32 first (both the GPU path and the
    oracle then see identical, exactly representable inputs).
    """
    if count < 1:
        raise ValueError("count must be >= 1")
    spec = spec or SyntheticSpec()
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-spec.extent, spec.extent, size=(count, 3))
    base = rng.uniform(spec.scale_range[0], spec.scale_range[1], size=count)
    ratios = rng.uniform(spec.anisotropy_range[0], spec.anisotropy_range[1], size=count)
    major = rng.integers(0, 3, size=count)
    scales = np.repeat(base[:, None], 3, axis=1)
    scales[np.arange(count), major] *= ratios
    quats = rng.normal(size=(count, 4))
    norms = np.linalg.norm(quats, axis=1)
    bad = norms < 1e-12
    quats[bad] = (1.0, 0.0, 0.0, 0.0)
    norms[bad] = 1.0
    quats /= norms[:, None]
    opac = rng.uniform(spec.opacity_range[0], spec.opacity_range[1], size=count)
    rgb = rng.uniform(0.0, 1.0, size=(count, 3))
    dc = (rgb - 0.5) / SH_C0
    k = (sh_degree + 1) ** 2
    sh = np.empty((count, k, 3))
    sh[:, 0, :] = dc
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, sh_rest_sigma, size=(count, k - 1, 3))
    arrs = SceneArrays(centers, scales, quats, opac, sh)
    if float32:
        arrs = SceneArrays(*(np.asarray(a, dtype=np.float32).astype(np.float64) for a in arrs))
    return arrs


def generate_synthetic(seed: int, count: int, spec: SyntheticSpec | None = None) -> Scene:
    """Deterministic degree-0 scene, value-identical to the reference's."""
    a = synthetic_arrays(seed, count, spec)
    gs = [Gaussian3D(a.centers[i], a.scales[i], a.rotations[i], a.opacities[i], a.sh[i])
          for i in range(count)]
    return Scene(gaussians=gs, sh_degree=0)


def _exact_in_f32(a: np.ndarray) -> bool:
    if a.dtype == np.float32:
        return True
    if a.dtype != np.float64:
        return False
    with np.errstate(over="ignore", invalid="ignore"):
        return bool(np.array_equal(a.astype(np.float32).astype(np.float64), a, equal_nan=True))


def _aligned(t, align: int = 16):
    return t if t.data_ptr() % align == 0 else t.clone()


class DeviceScene:
    """SoA scene resident on the GPU (what ``adr_scene`` points at).

    Arrays: centers (N,3), scales (N,3), rotations (N,4) wxyz, opacities (N,),
    sh (N,K,3); all fp32 or all fp64, contiguous, on one CUDA device.
    """

    def __init__(self, centers, scales, rotations, opacities, sh, sh_degree: int):
        import torch

        ts = [centers, scales, rotations, opacities, sh]
        dt = ts[0].dtype
        if dt not in (torch.float32, torch.float64):
            raise ValueError("scene tensors must be float32 or float64")
        if any(t.dtype != dt for t in ts):
            raise ValueError("scene tensors must share one dtype")
        if not 0 <= sh_degree <= MAX_SH_DEGREE:
            raise SceneValidationError(f"sh_degree {sh_degree} outside 0..{MAX_SH_DEGREE}")
        n = ts[3].numel()
        k = (sh_degree + 1) ** 2
        shapes = [(n, 3), (n, 3), (n, 4), (n,), (n, k, 3)]
        # contiguous and 16-byte aligned (the preprocess stages the SH slab
        # with 16-byte vector loads): an offset view is copied
        self.centers, self.scales, self.rotations, self.opacities, self.sh = (
            _aligned(t.reshape(s).contiguous()) for t, s in zip(ts, shapes))
        self.sh_degree = int(sh_degree)

    def __len__(self) -> int:
        return self.opacities.numel()

    @property
    def device(self):
        return self.centers.device

    @classmethod
    def from_arrays(cls, arrays, sh_degree: int, device="cuda", dtype=None) -> "DeviceScene":
        """Upload host arrays.  ``dtype=None`` picks float32 when every value
        is exactly representable in it (the fp32 -> fp64 promotion inside the
        kernel then reproduces the fp64 inputs bit for bit, at half the
        bytes), else float64."""
        import torch

        arrays = [np.asarray(a) for a in arrays]
        if dtype is None:
            dtype = torch.float32 if all(_exact_in_f32(a) for a in arrays) else torch.float64
        np_dt = np.float32 if dtype == torch.float32 else np.float64
        return cls(*(torch.from_numpy(np.ascontiguousarray(a, dtype=np_dt)).to(device)
                     for a in arrays), sh_degree=sh_degree)

    @classmethod
    def from_scene(cls, scene, device="cuda", dtype=None) -> "DeviceScene":
        """From a Scene (ours or the reference's, fp64) or a DeviceScene."""
        if isinstance(scene, DeviceScene):
            return scene.to(device)
        if isinstance(scene, SceneArrays):   # degree from the (N, (d+1)^2, 3) SH block
            deg = int(round(np.sqrt(scene.sh.shape[1]))) - 1
            if (deg + 1) ** 2 != scene.sh.shape[1]:
                raise ValueError(f"sh has {scene.sh.shape[1]} coefficients, not a square (d+1)^2")
            return cls.from_arrays(scene, deg, device, dtype)
        return cls.from_arrays(scene.as_arrays(), int(scene.sh_degree), device, dtype)

    def to(self, device) -> "DeviceScene":
        if self.centers.device == device or str(self.centers.device) == str(device):
            return self
        return DeviceScene(*(t.to(device) for t in (self.centers, self.scales, self.rotations,
                                                    self.opacities, self.sh)), self.sh_degree)

    def pin_memory(self) -> "DeviceScene":
        return DeviceScene(*(t.pin_memory() for t in (self.centers, self.scales, self.rotations,
                                                      self.opacities, self.sh)), self.sh_degree)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.centers, self.scales,
                                                          self.rotations, self.opacities, self.sh))

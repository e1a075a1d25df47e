"""Stage 1 — preprocess (sb/projection.py), on the GPU.

``preprocess`` keeps the reference signature and error behaviour
(sb/projection.py:291-304) and returns a ``Projection`` whose fields are CUDA
tensors with the reference's shapes and dtypes; ``Projection.to_numpy()``
gives the reference's numpy layout.  The math runs in
``adr_preprocess`` (csrc/adr_preprocess.cu): fp64, reference evaluation order.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .scene import DeviceScene

# Constants of sb/projection.py:33-43.
ALPHA_LOW = 1.0 / 255.0
COV_DILATION = 0.3
BASE_RADIUS_MULTIPLIER = 3.0
FOV_CLAMP_FACTOR = 1.3


class CullingMode(enum.Enum):
    """sb/projection.py:46-49."""

    BASELINE = "baseline"
    CIRCLE = "circle"
    AABB = "aabb"


_ARRAY_FIELDS = ("valid", "mean2d", "cov2d", "conic", "depth", "color", "opacity", "lambda_max",
                 "ext_x", "ext_y")


@dataclass(eq=False)
class Projection:
    """Batched preprocessing output, index-aligned with the scene
    (sb/projection.py:86-112); arrays are CUDA tensors."""

    mode: CullingMode
    alpha_low: float
    valid: object        # (N,) bool
    mean2d: object       # (N, 2) float32
    cov2d: object        # (N, 3) float32: sxx, syy, sxy
    conic: object        # (N, 3) float32: a, b, c
    depth: object        # (N,) float32
    color: object        # (N, 3) float32
    opacity: object      # (N,) float32
    lambda_max: object   # (N,) float32
    ext_x: object        # (N,) int32
    ext_y: object        # (N,) int32

    def __len__(self) -> int:
        return int(self.valid.shape[0])

    @property
    def culled_count(self) -> int:
        return int((~self.valid).sum().item())

    def struct(self, contiguous: bool = True) -> _lib.Projection_t:
        """C view of the arrays.  The library reads and writes them as
        contiguous SoA, so strided fields (a fused frame's views into its
        render record) are passed as contiguous copies, kept alive on the
        object; ``contiguous=False`` passes the raw pointers (the frame call,
        which does not touch those fields)."""
        p = _lib.Projection_t()
        keep = []
        for name in _ARRAY_FIELDS:
            t = getattr(self, name)
            if contiguous and not t.is_contiguous():
                t = t.contiguous()
                keep.append(t)
            setattr(p, "d_" + name, _lib.ptr(t))
        self._struct_copies = keep
        return p

    def to_numpy(self) -> dict:
        return {name: getattr(self, name).cpu().numpy() for name in _ARRAY_FIELDS}

    def clone(self) -> "Projection":
        """Contiguous copies of every array (also of record-backed views)."""
        import torch

        return Projection(mode=self.mode, alpha_low=self.alpha_low,
                          **{name: getattr(self, name).clone(memory_format=torch.contiguous_format)
                             for name in _ARRAY_FIELDS})

    @classmethod
    def empty(cls, n: int, mode, alpha_low, device) -> "Projection":
        import torch

        f32 = dict(dtype=torch.float32, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        return cls(mode=CullingMode(mode), alpha_low=alpha_low,
                   valid=torch.empty(n, dtype=torch.bool, device=device),
                   mean2d=torch.empty((n, 2), **f32), cov2d=torch.empty((n, 3), **f32),
                   conic=torch.empty((n, 3), **f32), depth=torch.empty(n, **f32),
                   color=torch.empty((n, 3), **f32), opacity=torch.empty(n, **f32),
                   lambda_max=torch.empty(n, **f32), ext_x=torch.empty(n, **i32),
                   ext_y=torch.empty(n, **i32))

    @classmethod
    def from_numpy(cls, arrays: dict, mode, alpha_low, device="cuda") -> "Projection":
        """Upload a reference-layout projection (e.g. a reference Projection's
        arrays) so the later GPU stages can consume it."""
        import torch

        kw = {}
        for name in _ARRAY_FIELDS:
            a = arrays[name] if isinstance(arrays, dict) else getattr(arrays, name)
            kw[name] = torch.as_tensor(np.ascontiguousarray(a)).to(device)
        return cls(mode=CullingMode(mode), alpha_low=alpha_low, **kw)


def as_device_scene(scene, device=None) -> DeviceScene:
    """The scene on a CUDA device: a CUDA DeviceScene as is, a host one (e.g.
    pinned) uploaded, anything else converted (DeviceScene.from_scene)."""
    import torch

    if device is None:
        on_cuda = isinstance(scene, DeviceScene) and scene.device.type == "cuda"
        device = scene.device if on_cuda else torch.device("cuda")
    return DeviceScene.from_scene(scene, device=device)


def scene_struct(ds: DeviceScene) -> _lib.Scene_t:
    import torch

    s = _lib.Scene_t()
    s.d_centers, s.d_scales, s.d_rotations = (_lib.ptr(ds.centers), _lib.ptr(ds.scales),
                                              _lib.ptr(ds.rotations))
    s.d_opacities, s.d_sh = _lib.ptr(ds.opacities), _lib.ptr(ds.sh)
    s.n = len(ds)
    s.sh_degree = ds.sh_degree
    s.dtype = _lib.ADR_F32 if ds.centers.dtype == torch.float32 else _lib.ADR_F64
    return s


def _validate(alpha_low, dilation, mode) -> CullingMode:
    if not 0.0 < alpha_low < 1.0:
        raise ValueError("alpha_low must lie in (0, 1)")
    if dilation < 0:
        raise ValueError("dilation must be non-negative")
    return CullingMode(mode)


def preprocess(scene, cam, mode: CullingMode = CullingMode.AABB, alpha_low: float = ALPHA_LOW,
               dilation: float = COV_DILATION, threads: int = 1) -> Projection:
    """Project every Gaussian and compute its culling extent
    (sb/projection.py:291-334).  ``threads`` is accepted for signature
    compatibility; the GPU result never depends on it."""
    import torch

    mode = _validate(alpha_low, dilation, mode)
    ds = as_device_scene(scene)
    n = len(ds)
    out = Projection.empty(n, mode, alpha_low, ds.device)
    if n:
        with torch.cuda.device(ds.device):
            st = torch.cuda.current_stream()
            _lib.check(_lib.lib().adr_preprocess(
                scene_struct(ds), _lib.camera_struct(cam), _lib.MODE_CODES[mode.value],
                float(alpha_low), float(dilation), out.struct(), _lib.stream_handle(st)))
    return out


__all__ = ["ALPHA_LOW", "COV_DILATION", "BASE_RADIUS_MULTIPLIER", "FOV_CLAMP_FACTOR",
           "CullingMode", "Projection", "preprocess", "as_device_scene", "scene_struct"]


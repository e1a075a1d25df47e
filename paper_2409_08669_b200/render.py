"""Stage 6 — blending + load map (sb/render.py), on the GPU.

``render`` keeps the reference signature, checks and exceptions
(sb/render.py:128-188); the per-tile blend runs in ``adr_render``
(csrc/adr_render.cu) with the exact fp32 recurrence of the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .errors import InternalError
from .projection import Projection
from .tiling import TileGrid, TilePairList

# Constants of sb/render.py:31-36.
ALPHA_CLAMP = 0.99
TERMINATION_THRESHOLD = 1e-4


@dataclass(eq=False)
class Image:
    """Row-major float32 RGB image in [0, 1] (sb/render.py:40-46); CUDA tensor."""

    width: int
    height: int
    pixels: object  # (height, width, 3) float32


@dataclass(eq=False)
class LoadMap:
    """Per-pixel count of composited Gaussians (sb/render.py:49-55); CUDA tensor."""

    width: int
    height: int
    counts: object  # (height, width) int32


def _check_consistency(proj: Projection, pairs: TilePairList, grid: TileGrid, cam) -> None:
    """sb/render.py:174-188."""
    if pairs.tile_ranges is None:
        raise InternalError("tile ranges were not identified")
    if tuple(pairs.tile_ranges.shape) != (grid.n_tiles, 2):
        raise InternalError("tile ranges do not match the grid")
    if len(pairs.keys) != len(pairs.gaussian_indices):
        raise InternalError("pair arrays are not parallel")
    if len(pairs.keys) and int(pairs.gaussian_indices.max().item()) >= len(proj):
        raise InternalError("pair references a Gaussian outside the projection")
    if (grid.width, grid.height) != (cam.width, cam.height):
        raise InternalError("grid does not match the camera resolution")
    if len(pairs.keys):
        r = pairs.tile_ranges
        if int(r[0, 0].item()) != 0 or int(r[-1, 1].item()) != len(pairs.keys):
            raise InternalError("tile ranges do not partition the pair list")


def render(proj: Projection, pairs: TilePairList, grid: TileGrid, cam, alpha_low: float,
           term_threshold: float = TERMINATION_THRESHOLD, threads: int = 1):
    """Render every tile's span into an image and load map (sb/render.py:128-171)."""
    import torch

    _check_consistency(proj, pairs, grid, cam)
    dev = proj.valid.device
    h, w = int(cam.height), int(cam.width)
    pixels = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    counts = torch.empty((h, w), dtype=torch.int32, device=dev)
    gidx = pairs.gaussian_indices.to(device=dev, dtype=torch.int64).contiguous()
    ranges = pairs.tile_ranges.to(device=dev, dtype=torch.int64).contiguous()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().adr_render(
            proj.struct(), len(proj), _lib.ptr(gidx), gidx.numel(), _lib.ptr(ranges),
            _lib.camera_struct(cam), float(alpha_low), float(term_threshold), _lib.ptr(pixels),
            _lib.ptr(counts), None, None, 0,
            _lib.stream_handle(torch.cuda.current_stream())))
    return Image(width=w, height=h, pixels=pixels), LoadMap(width=w, height=h, counts=counts)

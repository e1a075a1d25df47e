"""Brute-force reference renderer on the GPU (sb/oracle.py:23-83; SURVEY.md
§8f row 3).

``render_reference`` bypasses the tile binning entirely: a BASELINE-mode
preprocess, one global stable sort of the valid Gaussians by (float32 depth
bits, index), and per tile a walk over every Gaussian whose footprint
rectangle overlaps the tile (the reference's own interval test), blended
with the exact scalar recurrence.  Its image and load map must equal
``run_pipeline``'s bit for bit, which makes it a large-N self-check of stages
2-5 that needs no CPU oracle (csrc/adr_refrender.cu).
"""

from __future__ import annotations

from . import _lib
from .projection import ALPHA_LOW, CullingMode, as_device_scene, preprocess
from .render import TERMINATION_THRESHOLD, Image, LoadMap
from .tiling import TILE_SIZE


def grid_right(width: int) -> float:
    """Pixel coordinate of the right edge of the rightmost tile (sb/oracle.py:81-83)."""
    return float(-(-width // TILE_SIZE) * TILE_SIZE)


def render_reference(scene, cam, alpha_low: float = ALPHA_LOW,
                     term_threshold: float = TERMINATION_THRESHOLD):
    """(Image, LoadMap) without tiling (sb/oracle.py:23-78), on the GPU."""
    import torch

    ds = as_device_scene(scene)
    proj = preprocess(ds, cam, mode=CullingMode.BASELINE, alpha_low=alpha_low)
    n = len(ds)
    dev = ds.device
    pixels = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
    load = torch.empty((cam.height, cam.width), dtype=torch.int32, device=dev)
    L = _lib.lib()
    scratch = torch.empty(int(L.adr_render_reference_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream()
        _lib.check(L.adr_render_reference(proj.struct(), n, _lib.camera_struct(cam), float(alpha_low),
                                          float(term_threshold), _lib.ptr(pixels), _lib.ptr(load),
                                          _lib.ptr(scratch), scratch.numel(), _lib.stream_handle(st)))
    return Image(cam.width, cam.height, pixels), LoadMap(cam.width, cam.height, load)

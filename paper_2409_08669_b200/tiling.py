"""Stages 2-5 — tile binning (sb/tiling.py), on the GPU.

Same function names, arguments and exceptions as the reference; arrays are
CUDA tensors (keys: torch.uint64 bit patterns, gaussian_indices: int64).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CapacityError, InternalError
from .projection import Projection

TILE_SIZE = 16


@dataclass(frozen=True)
class TileGrid:
    """16x16-pixel tiles over the image; edge tiles may be partial (sb/tiling.py:25-48)."""

    width: int
    height: int
    tile_size: int = TILE_SIZE

    def __post_init__(self) -> None:
        if self.width < 1 or self.height < 1:
            raise ValueError("grid dimensions must be positive")
        if self.tiles_x * self.tiles_y >= 2 ** 32:
            raise CapacityError("tile count does not fit the 32-bit key field")

    @property
    def tiles_x(self) -> int:
        return -(-self.width // self.tile_size)

    @property
    def tiles_y(self) -> int:
        return -(-self.height // self.tile_size)

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y


@dataclass(frozen=True)
class TileRect:
    """Half-open tile rectangle [x0, x1) x [y0, y1) (sb/tiling.py:52-62)."""

    x0: int
    y0: int
    x1: int
    y1: int

    @property
    def count(self) -> int:
        return max(0, self.x1 - self.x0) * max(0, self.y1 - self.y0)


@dataclass(eq=False)
class TilePairList:
    """Sorted (key, Gaussian index) pairs plus per-tile spans (sb/tiling.py:66-74)."""

    keys: object                    # (P,) uint64, ascending
    gaussian_indices: object        # (P,) int64 (int32 from the fused frame)
    tile_ranges: object = None      # (n_tiles, 2) int64

    def __len__(self) -> int:
        return int(self.keys.shape[0])

    def to_numpy(self) -> dict:
        out = {"keys": self.keys.cpu().numpy().astype(np.uint64, copy=False),
               "gaussian_indices": self.gaussian_indices.cpu().numpy().astype(np.int64, copy=False)}
        if self.tile_ranges is not None:
            out["tile_ranges"] = self.tile_ranges.cpu().numpy()
        return out


def _device_of(t):
    return t.device


def _stream():
    import torch

    return _lib.stream_handle(torch.cuda.current_stream())


def _tensor(x, dtype, device):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x)), dtype=dtype).to(device)


def tiles_touched(pg, grid: TileGrid) -> TileRect:
    """Tile rectangle of one projected Gaussian (sb/tiling.py:102-108).

    A scalar helper of the reference's unit tests; evaluated on the host with
    the same fp64 floor/clip expression the touched-count kernel uses."""
    mx, my = (float(v) for v in np.asarray(pg.mean2d, dtype=np.float64).reshape(2))
    ex, ey = float(pg.extent.rx), float(pg.extent.ry)
    ts = grid.tile_size
    clip = lambda v, hi: min(max(v, 0.0), float(hi))
    x0 = int(clip(np.floor((mx - ex) / ts), grid.tiles_x))
    x1 = int(clip(np.floor((mx + ex) / ts) + 1, grid.tiles_x))
    y0 = int(clip(np.floor((my - ey) / ts), grid.tiles_y))
    y1 = int(clip(np.floor((my + ey) / ts) + 1, grid.tiles_y))
    return TileRect(x0=x0, y0=y0, x1=max(x1, x0), y1=max(y1, y0))


def touched_counts(proj: Projection, grid: TileGrid):
    """Per-Gaussian touched-tile counts, 0 for culled/off-screen (sb/tiling.py:111-114)."""
    import torch

    n = len(proj)
    dev = _device_of(proj.valid)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    if n:
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().adr_touched_counts(proj.struct(), n, grid.tiles_x, grid.tiles_y,
                                                     _lib.ptr(counts), _stream()))
    return counts


def inclusive_sum(counts, device=None):
    """Inclusive prefix sum, int64; CapacityError past INT64_MAX (sb/tiling.py:117-122)."""
    import torch

    if isinstance(counts, torch.Tensor):
        dev = counts.device if counts.is_cuda else (device or torch.device("cuda"))
        c = counts.to(device=dev, dtype=torch.int64).contiguous()
    else:
        arr = [int(v) for v in np.asarray(counts, dtype=object).reshape(-1)]
        if any(v > 2 ** 63 - 1 or v < -(2 ** 63) for v in arr):
            raise CapacityError("pair count overflows the 64-bit index type")
        dev = device or torch.device("cuda")
        c = torch.tensor(arr, dtype=torch.int64, device=dev) if arr else \
            torch.empty(0, dtype=torch.int64, device=dev)
    n = c.numel()
    out = torch.empty(n, dtype=torch.int64, device=dev)
    if n == 0:
        return out
    L = _lib.lib()
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    scratch = torch.empty(L.adr_inclusive_sum_scratch_bytes(n), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.check(L.adr_inclusive_sum(_lib.ptr(c), n, _lib.ptr(out), _lib.ptr(flag),
                                       _lib.ptr(scratch), scratch.numel(), _stream()))
    if int(flag.item()):
        raise CapacityError("pair count overflows the 64-bit index type")
    return out


def duplicate_with_keys(proj: Projection, offsets, grid: TileGrid):
    """One (key, Gaussian index) entry per touched tile (sb/tiling.py:125-156)."""
    import torch

    dev = _device_of(proj.valid)
    offsets = _tensor(offsets, torch.int64, dev)
    if tuple(offsets.shape) != (len(proj),):
        raise InternalError("offsets do not match the projection")
    total = int(offsets[-1].item()) if offsets.numel() else 0
    keys = torch.empty(total, dtype=torch.uint64, device=dev)
    gidx = torch.empty(total, dtype=torch.int64, device=dev)
    if total:
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().adr_duplicate_with_keys(
                proj.struct(), len(proj), _lib.ptr(offsets), grid.tiles_x, grid.tiles_y,
                _lib.ptr(keys), _lib.ptr(gidx), _stream()))
    return keys, gidx


def _key_bits(keys) -> int:
    import torch

    if keys.numel() == 0:
        return 0
    s = keys.view(torch.int64)
    if bool((s < 0).any().item()):
        return 64
    return int(s.max().item()).bit_length()


def sort_pairs(keys, gaussian_indices, end_bit: int | None = None) -> TilePairList:
    """Stable ascending sort by key; ties keep emission order (sb/tiling.py:159-164)."""
    import torch

    if isinstance(keys, torch.Tensor):
        dev = keys.device
        k = keys.contiguous()
        if k.dtype != torch.uint64:
            k = k.to(torch.int64).view(torch.uint64)
    else:
        dev = torch.device("cuda")
        k = torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))).to(dev)
    v = _tensor(gaussian_indices, torch.int64, dev)
    if k.numel() != v.numel():
        raise InternalError("keys and gaussian_indices must be parallel")
    p = k.numel()
    ko = torch.empty_like(k)
    vo = torch.empty_like(v)
    if p:
        L = _lib.lib()
        bits = _key_bits(k) if end_bit is None else int(end_bit)
        scratch = torch.empty(L.adr_sort_pairs_scratch_bytes(p), dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(L.adr_sort_pairs(_lib.ptr(k), _lib.ptr(v), p, bits, _lib.ptr(ko),
                                        _lib.ptr(vo), _lib.ptr(scratch), scratch.numel(),
                                        _stream()))
    return TilePairList(keys=ko, gaussian_indices=vo)


def identify_tile_ranges(sorted_keys, grid: TileGrid):
    """Per-tile half-open spans; empty tiles get (k, k) (sb/tiling.py:167-177)."""
    import torch

    if isinstance(sorted_keys, torch.Tensor):
        dev = sorted_keys.device
        k = sorted_keys.contiguous()
        if k.dtype != torch.uint64:
            k = k.to(torch.int64).view(torch.uint64)
    else:
        dev = torch.device("cuda")
        k = torch.from_numpy(np.ascontiguousarray(np.asarray(sorted_keys, dtype=np.uint64))).to(dev)
    ranges = torch.empty((grid.n_tiles, 2), dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().adr_identify_tile_ranges(_lib.ptr(k), k.numel(), grid.n_tiles,
                                                       _lib.ptr(ranges), _lib.ptr(err), _stream()))
    e = int(err.item())
    if e == 1:
        raise InternalError("keys are not sorted")
    if e == 2:
        raise InternalError("key references a tile outside the grid")
    return ranges


def build_pairs(proj: Projection, grid: TileGrid) -> TilePairList:
    """Stages 2-5 in sequence (sb/tiling.py:180-187)."""
    counts = touched_counts(proj, grid)
    offsets = inclusive_sum(counts)
    keys, gidx = duplicate_with_keys(proj, offsets, grid)
    end_bit = 32 + max(1, (grid.n_tiles - 1).bit_length())
    pairs = sort_pairs(keys, gidx, end_bit=end_bit)
    pairs.tile_ranges = identify_tile_ranges(pairs.keys, grid)
    return pairs

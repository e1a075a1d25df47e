"""View-sharded multi-GPU rendering.

Views are independent units: the scene is replicated on every rank, view k of
a V-view batch goes to rank floor(k * R / V) (contiguous slices), each rank
renders its slice back to back on its own GPU, and the only collective is the
final gather of frames (+ a fixed-size stats vector) to rank 0 over NCCL.
Per-view outputs therefore equal single-GPU renders bit for bit.
"""

from __future__ import annotations

import math

import numpy as np

from .scene import Camera


def orbit_cameras(n_views: int, width: int, height: int, radius: float = 2.6,
                  fov_y_deg: float = 60.0, background=(0.0, 0.0, 0.0), height_y: float = 0.0):
    """Camera k at (r sin t, y, -r cos t), t = 2 pi k / V, looking at the origin."""
    cams = []
    for k in range(n_views):
        t = 2.0 * math.pi * k / n_views
        cams.append(Camera.from_lookat((radius * math.sin(t), height_y, -radius * math.cos(t)),
                                       (0.0, 0.0, 0.0), fov_y_deg=fov_y_deg, width=width,
                                       height=height, background=background))
    return cams


def shard_views(n_views: int, world: int, rank: int) -> range:
    """Contiguous slice of views owned by `rank`: view k -> floor(k * world / n_views)."""
    if n_views < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    lo = -(-rank * n_views // world)
    hi = -(-(rank + 1) * n_views // world)
    return range(lo, hi)


def owner_of(view: int, n_views: int, world: int) -> int:
    return view * world // n_views


STATS_FIELDS = ("pairs", "culled", "load_sum", "load_sum_sq", "load_min", "load_max")


def gather_frames(frames, stats, n_views: int, group=None, dst: int = 0):
    """Gather per-view frames to `dst`.

    frames: (local_views, H, W, 4) float32 (RGB + load as float bits) on this
    rank's device; stats: (local_views, 6) int64.  Slices can be ragged
    (V not divisible by R): every rank pads to ceil(V/R) rows so one
    all_gather_into_tensor moves everything; rank `dst` then drops the padding
    and returns (V, H, W, 4), (V, 6) in view order (others return None).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_views // world)
    h, w = frames.shape[1], frames.shape[2]
    pad_f = torch.zeros((per, h, w, 4), dtype=frames.dtype, device=frames.device)
    pad_s = torch.zeros((per, len(STATS_FIELDS)), dtype=torch.int64, device=frames.device)
    pad_f[: frames.shape[0]] = frames
    pad_s[: stats.shape[0]] = stats
    all_f = torch.empty((world * per, h, w, 4), dtype=frames.dtype, device=frames.device)
    all_s = torch.empty((world * per, len(STATS_FIELDS)), dtype=torch.int64, device=frames.device)
    dist.all_gather_into_tensor(all_f, pad_f, group=group)
    dist.all_gather_into_tensor(all_s, pad_s, group=group)
    if rank != dst:
        return None, None
    rows = np.concatenate([np.arange(r * per, r * per + len(shard_views(n_views, world, r)))
                           for r in range(world)])
    idx = torch.as_tensor(rows, device=frames.device)
    return all_f.index_select(0, idx), all_s.index_select(0, idx)


def pack_frame(pixels, load):
    """(H,W,3) float32 + (H,W) int32 -> (H,W,4) float32 (load stored as bits)."""
    import torch

    return torch.cat([pixels, load.view(torch.float32).unsqueeze(-1)], dim=-1)


def unpack_frame(frame):
    import torch

    return frame[..., :3], frame[..., 3].contiguous().view(torch.int32)

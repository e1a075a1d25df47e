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


def broadcast_scene(scene, n: int, sh_degree: int, device, dtype=None, group=None, src: int = 0):
    """Replicate a scene from rank `src` on every rank (load
    once, broadcast N·(44 + 12K) bytes at fp32).  `scene` is the source
    rank's DeviceScene (ignored elsewhere); every rank passes the same N and
    SH degree and gets a DeviceScene of its own on `device`."""
    import torch
    import torch.distributed as dist

    from .scene import DeviceScene

    dtype = dtype or (scene.centers.dtype if scene is not None else torch.float32)
    k = (sh_degree + 1) ** 2
    shapes = [(n, 3), (n, 3), (n, 4), (n,), (n, k, 3)]
    if dist.get_rank(group) == src:
        ts = [t.to(device=device, dtype=dtype).contiguous() for t in
              (scene.centers, scene.scales, scene.rotations, scene.opacities, scene.sh)]
    else:
        ts = [torch.empty(sh, dtype=dtype, device=device) for sh in shapes]
    for t in ts:
        dist.broadcast(t, src=src, group=group)
    return DeviceScene(*ts, sh_degree=sh_degree)


def pack_frame(pixels, load):
    """(H,W,3) float32 + (H,W) int32 -> (H,W,4) float32 (load stored as bits)."""
    import torch

    return torch.cat([pixels, load.view(torch.float32).unsqueeze(-1)], dim=-1)


def unpack_frame(frame):
    import torch

    return frame[..., :3], frame[..., 3].contiguous().view(torch.int32)


class ViewRenderer:
    """Renders a batch of cameras of one resident scene with several views in
    flight (BASELINE configs[3]/[4]).

    Each in-flight slot owns a ``Rasterizer`` (persistent buffers) and a CUDA
    stream; view i renders in slot i mod K, so frames of different views
    overlap on the GPU while every frame stays a fixed kernel sequence.
    Results are copied into batch tensors on the slot's stream; a view whose
    pairs exceed its slot's capacity is re-rendered with larger buffers, so
    every output equals a single-view ``run_pipeline`` bit for bit.
    """

    def __init__(self, scene, width: int, height: int, in_flight: int = 4, device=None):
        import torch

        from .pipeline import Rasterizer
        from .projection import as_device_scene

        self.scene = as_device_scene(scene, device)
        self.device = self.scene.device
        self.width, self.height = int(width), int(height)
        k = max(1, int(in_flight))
        self.slots = [Rasterizer(self.width, self.height, len(self.scene), device=self.device, timing=False)
                      for _ in range(k)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(k)]

    def render(self, cams, mode="aabb", alpha_low=None):
        """-> (pixels (V,H,W,3) f32, load (V,H,W) i32, stats (V, 6) i64 in
        STATS_FIELDS order) as CUDA tensors."""
        import torch

        from .projection import ALPHA_LOW

        alpha_low = ALPHA_LOW if alpha_low is None else alpha_low
        v = len(cams)
        dev = self.device
        pixels = torch.empty((v, self.height, self.width, 3), dtype=torch.float32, device=dev)
        load = torch.empty((v, self.height, self.width), dtype=torch.int32, device=dev)
        stats = torch.empty((v, len(STATS_FIELDS)), dtype=torch.int64, device=dev)
        k = len(self.slots)
        main = torch.cuda.current_stream(dev)
        ev = torch.cuda.Event()
        ev.record(main)
        for st in self.streams:
            st.wait_event(ev)

        def one(i):
            r, st = self.slots[i % k], self.streams[i % k]
            with torch.cuda.stream(st):
                r.launch(self.scene, cams[i], mode, alpha_low, stream=st)
                pixels[i].copy_(r.pixels, non_blocking=True)
                load[i].copy_(r.load, non_blocking=True)
                stats[i, 0:2].copy_(r.counters[0:2], non_blocking=True)
                stats[i, 2:4].copy_(r.stats[0:2], non_blocking=True)
                mm = r.stats[2:3]   # packed (min, max) int32 pair
                stats[i, 4] = mm & 0xFFFFFFFF
                stats[i, 5] = (mm >> 32) & 0xFFFFFFFF

        for i in range(v):
            one(i)
        for st in self.streams:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)
        torch.cuda.synchronize(dev)
        # views that overflowed their slot: grow that slot, render again
        caps = torch.tensor([self.slots[i % k].cap for i in range(v)], dtype=torch.int64)
        over = (stats[:, 0].cpu() > caps).nonzero().flatten().tolist()
        for i in over:
            slot = self.slots[i % k]
            slot.fit_capacity(int(stats[i, 0].item() * 1.25) + 1024)
            one(i)
            torch.cuda.synchronize(dev)
        # the min/max halves are signed int32
        for c in (4, 5):
            col = stats[:, c]
            stats[:, c] = torch.where(col >= (1 << 31), col - (1 << 32), col)
        return pixels, load, stats


def render_views_sharded(scene, cams, in_flight: int = 4, group=None, dst: int = 0):
    """Multi-GPU view-sharded rendering: this rank renders its contiguous
    slice of ``cams`` (``shard_views``) with a ``ViewRenderer`` and the frames
    plus stats are gathered to ``dst`` (``gather_frames``).  Returns
    (pixels (V,H,W,3), load (V,H,W), stats (V,6)) on ``dst``, (None, None,
    None) elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = [cams[i] for i in shard_views(len(cams), world, rank)]
    w, h = cams[0].width, cams[0].height
    vr = ViewRenderer(scene, w, h, in_flight)
    if mine:
        px, ld, st = vr.render(mine)
    else:
        import torch

        px = torch.empty((0, h, w, 3), dtype=torch.float32, device=vr.device)
        ld = torch.empty((0, h, w), dtype=torch.int32, device=vr.device)
        st = torch.empty((0, len(STATS_FIELDS)), dtype=torch.int64, device=vr.device)
    frames = pack_frame(px, ld) if len(mine) else px.new_empty((0, h, w, 4))
    all_f, all_s = gather_frames(frames, st, len(cams), group=group, dst=dst)
    if all_f is None:
        return None, None, None
    p, l = unpack_frame(all_f)
    return p.contiguous(), l, all_s

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


def _wire(t, group):
    """NCCL moves device tensors; gloo only host tensors."""
    import torch.distributed as dist

    return t.cpu() if (t.is_cuda and dist.get_backend(group) == "gloo") else t


class FrameGather:
    """Gathers the frames of a V-view batch to rank ``dst`` with point-to-point
    transfers that overlap the rendering (NCCL moves frames and
    stats only, to one rank).

    Each view's payload is one float32 buffer: (H, W, 4) RGB + load (load as
    int32 bits) followed by the 6 int64 stats as 12 float32 words.  A rank
    that rendered view v calls ``send(v, ...)`` right after the frame was
    enqueued (on the frame's stream, so the transfer waits for exactly that
    frame); ``dst`` posts one receive per remote view in ``begin()``;
    ``finish()`` makes the current stream wait for every transfer and returns
    (pixels (V,H,W,3), load (V,H,W), stats (V,6)) views of the batch buffer on
    ``dst`` (None elsewhere).  Ranks send in view order and ``dst`` receives in
    view order, so transfers pair up on every backend (NCCL or gloo).
    """

    def __init__(self, n_views: int, height: int, width: int, device, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist

        self.v, self.h, self.w = int(n_views), int(height), int(width)
        self.group, self.dst = group, dst
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device)
        self.words = self.h * self.w * 4 + 2 * len(STATS_FIELDS)
        mine = shard_views(self.v, self.world, self.rank)
        self.mine = list(mine)
        rows = self.v if self.rank == dst else len(self.mine)
        self.buf = torch.empty((rows, self.words), dtype=torch.float32, device=self.device)
        self._works = []

    def _row(self, view: int) -> int:
        return view if self.rank == self.dst else view - self.mine[0]

    def begin(self) -> None:
        """Post the receives of this batch (dst only)."""
        import torch.distributed as dist

        self._works = []
        if self.rank != self.dst:
            return
        self._host = {}
        for view in range(self.v):
            src = owner_of(view, self.v, self.world)
            if src == self.dst:
                continue
            t = _wire(self.buf[view], self.group)
            if t is not self.buf[view]:
                self._host[view] = t
            self._works.append((dist.irecv(t, src=src, group=self.group), t))

    def send(self, view: int, pixels, load, stats) -> None:
        """Pack one rendered view (enqueued on the current stream) and ship it."""
        import torch
        import torch.distributed as dist

        row = self.buf[self._row(view)]
        hw4 = self.h * self.w * 4
        row[:hw4].view(self.h, self.w, 4).copy_(pack_frame(pixels, load))
        row[hw4:].view(torch.int64).copy_(stats.reshape(-1).to(torch.int64))
        if self.rank != self.dst:
            t = _wire(row, self.group)   # (a host copy on gloo: kept alive until finish)
            self._works.append((dist.isend(t, dst=self.dst, group=self.group), t))

    def finish(self):
        import torch

        for w, _ in self._works:
            w.wait()
        for view, t in getattr(self, "_host", {}).items():
            self.buf[view].copy_(t)
        self._works = []
        if self.rank != self.dst:
            return None, None, None
        hw4 = self.h * self.w * 4
        frames = self.buf[:, :hw4].view(self.v, self.h, self.w, 4)
        stats = self.buf[:, hw4:].contiguous().view(torch.int64)
        px, ld = unpack_frame(frames)
        return px, ld, stats


def gather_frames(frames, stats, n_views: int, group=None, dst: int = 0):
    """Gather per-view frames to `dst` (a gather, not an all-gather: only
    `dst` receives).

    frames: (local_views, H, W, 4) float32 (RGB + load as float bits) of this
    rank's contiguous view slice; stats: (local_views, 6) int64.  Slices may
    be ragged or empty.  Returns (V, H, W, 4), (V, 6) in view order on `dst`,
    (None, None) elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    h, w = frames.shape[1], frames.shape[2]
    fg = FrameGather(n_views, h, w, frames.device, group=group, dst=dst)
    fg.begin()
    for i, view in enumerate(shard_views(n_views, world, rank)):
        px, ld = unpack_frame(frames[i])
        fg.send(view, px, ld, stats[i])
    px, ld, st = fg.finish()
    if px is None:
        return None, None
    return pack_frame_batch(px, ld), st


def pack_frame_batch(px, ld):
    import torch

    return torch.cat([px, ld.view(torch.float32).unsqueeze(-1)], dim=-1)


_DTYPES = ("float32", "float64")


def broadcast_scene(scene, n: int, sh_degree: int, device, dtype=None, group=None, src: int = 0):
    """Replicate a scene from rank `src` on every rank (load
    once, broadcast N·(44 + 12K) bytes at fp32).  `scene` is the source
    rank's DeviceScene (ignored elsewhere).  The source first broadcasts a
    header (N, SH degree, dtype), so every rank allocates identical buffers
    whatever it passed; a mismatch with the caller's N / degree raises.
    Returns a DeviceScene on `device` on every rank."""
    import torch
    import torch.distributed as dist

    from .scene import DeviceScene

    is_src = dist.get_rank(group) == src
    if is_src:
        dt = dtype or scene.centers.dtype
        hdr = torch.tensor([len(scene), scene.sh_degree, _DTYPES.index(str(dt).split(".")[-1])],
                           dtype=torch.int64)
    else:
        hdr = torch.zeros(3, dtype=torch.int64)
    hdr_w = hdr.to(device) if dist.get_backend(group) == "nccl" else hdr
    dist.broadcast(hdr_w, src=src, group=group)
    n_src, deg_src, code = (int(v) for v in hdr_w.cpu().tolist())
    if (n_src, deg_src) != (int(n), int(sh_degree)):
        raise ValueError(f"broadcast_scene: source has N={n_src}, degree {deg_src}; "
                         f"this rank expected N={n}, degree {sh_degree}")
    dtype = getattr(torch, _DTYPES[code])
    k = (sh_degree + 1) ** 2
    shapes = [(n, 3), (n, 3), (n, 4), (n,), (n, k, 3)]
    if is_src:
        ts = [t.to(device=device, dtype=dtype).contiguous() for t in
              (scene.centers, scene.scales, scene.rotations, scene.opacities, scene.sh)]
    else:
        ts = [torch.empty(sh, dtype=dtype, device=device) for sh in shapes]
    for i, t in enumerate(ts):
        w = _wire(t, group)
        dist.broadcast(w, src=src, group=group)
        if w is not t:
            t.copy_(w)
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

    Views are taken in groups of ``batch_views`` (<= 8): one
    ``preprocess_views`` launch runs stage 1 of the whole group (the scene is
    read once), then each view's stages 2-6 run in its own ``Rasterizer``
    slot on one of ``in_flight`` CUDA streams, so frames of different views
    overlap on the GPU; two slot sets alternate, so group g+1's stage 1
    overlaps group g's binning and render.  ``batch_views=1``: every view is
    one whole-frame call, view i in slot i mod ``in_flight``.  Results are
    copied into batch tensors on the slot's stream; a view whose pairs exceed
    its slot's capacity is re-rendered with larger buffers, so every output
    equals a single-view ``run_pipeline`` bit for bit.
    """

    def __init__(self, scene, width: int, height: int, in_flight: int = 4, device=None,
                 batch_views: int = 8):
        import torch

        from .pipeline import MAX_BATCH_VIEWS
        from .projection import as_device_scene

        self.scene = as_device_scene(scene, device)
        self.device = self.scene.device
        self.width, self.height = int(width), int(height)
        k = max(1, int(in_flight))
        self.batch = max(1, min(int(batch_views), MAX_BATCH_VIEWS))
        self.slots = []
        self._grow(k if self.batch == 1 else self.batch)
        self.streams = [torch.cuda.Stream(self.device) for _ in range(k)]
        self.pre_streams = [torch.cuda.Stream(self.device) for _ in range(2)]

    def _grow(self, n_slots: int) -> None:
        from .pipeline import Rasterizer

        while len(self.slots) < n_slots:
            self.slots.append(Rasterizer(self.width, self.height, len(self.scene), device=self.device,
                                         timing=False))

    def render(self, cams, mode="aabb", alpha_low=None):
        """-> (pixels (V,H,W,3) f32, load (V,H,W) i32, stats (V, 6) i64 in
        STATS_FIELDS order) as CUDA tensors."""
        import torch

        from .pipeline import preprocess_views
        from .projection import ALPHA_LOW

        alpha_low = ALPHA_LOW if alpha_low is None else alpha_low
        v = len(cams)
        dev = self.device
        pixels = torch.empty((v, self.height, self.width, 3), dtype=torch.float32, device=dev)
        load = torch.empty((v, self.height, self.width), dtype=torch.int32, device=dev)
        stats = torch.empty((v, len(STATS_FIELDS)), dtype=torch.int64, device=dev)
        k = len(self.streams)
        main = torch.cuda.current_stream(dev)
        ev = torch.cuda.Event()
        ev.record(main)
        for st in self.streams + self.pre_streams:
            st.wait_event(ev)

        def copy_out(i, r):
            pixels[i].copy_(r.pixels, non_blocking=True)
            load[i].copy_(r.load, non_blocking=True)
            stats[i, 0:2].copy_(r.counters[0:2], non_blocking=True)
            stats[i, 2:4].copy_(r.stats[0:2], non_blocking=True)
            mm = r.stats[2:3]   # packed (min, max) int32 pair
            stats[i, 4] = mm & 0xFFFFFFFF
            stats[i, 5] = (mm >> 32) & 0xFFFFFFFF

        def one(i, r):   # a whole frame of view i in slot r
            st = self.streams[i % k]
            with torch.cuda.stream(st):
                r.launch(self.scene, cams[i], mode, alpha_low, stream=st)
                copy_out(i, r)

        slot_of = {}
        if self.batch == 1:
            for i in range(v):
                slot_of[i] = self.slots[i % k]
                one(i, slot_of[i])
        else:
            b = self.batch
            groups = [list(range(g, min(g + b, v))) for g in range(0, v, b)]
            n_sets = min(2, len(groups))
            self._grow(b * n_sets)
            pending = [[] for _ in range(n_sets)]
            for gi, grp in enumerate(groups):
                ss = gi % n_sets
                ps = self.pre_streams[ss]
                for e in pending[ss]:
                    ps.wait_event(e)
                sl = [self.slots[ss * b + q] for q in range(len(grp))]
                preprocess_views(self.scene, [cams[i] for i in grp], sl, mode, alpha_low, stream=ps)
                pe = torch.cuda.Event()
                pe.record(ps)
                used = []
                for q, i in enumerate(grp):
                    slot_of[i] = sl[q]
                    st = self.streams[i % k]
                    st.wait_event(pe)
                    with torch.cuda.stream(st):
                        sl[q].launch_post(self.scene, cams[i], mode, alpha_low, stream=st)
                        copy_out(i, sl[q])
                    if st not in used:
                        used.append(st)
                pending[ss] = []
                for st in used:
                    e = torch.cuda.Event()
                    e.record(st)
                    pending[ss].append(e)
        for st in self.streams + self.pre_streams:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)
        torch.cuda.synchronize(dev)
        # views that overflowed their slot: grow that slot, render the view again
        caps = torch.tensor([slot_of[i].cap for i in range(v)], dtype=torch.int64)
        over = (stats[:, 0].cpu() > caps).nonzero().flatten().tolist()
        for i in over:
            slot = slot_of[i]
            slot.fit_capacity(int(stats[i, 0].item() * 1.25) + 1024)
            one(i, slot)
            torch.cuda.synchronize(dev)
        # the min/max halves are signed int32
        for c in (4, 5):
            col = stats[:, c]
            stats[:, c] = torch.where(col >= (1 << 31), col - (1 << 32), col)
        return pixels, load, stats


def render_views_sharded(scene, cams, in_flight: int = 4, group=None, dst: int = 0, batch_views: int = 8):
    """Multi-GPU view-sharded rendering: this rank renders its contiguous
    slice of ``cams`` (``shard_views``) with a ``ViewRenderer`` and the frames
    plus stats are gathered to ``dst`` (``FrameGather``).  Returns
    (pixels (V,H,W,3), load (V,H,W), stats (V,6)) on ``dst``, (None, None,
    None) elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    views = list(shard_views(len(cams), world, rank))
    w, h = cams[0].width, cams[0].height
    vr = ViewRenderer(scene, w, h, in_flight, batch_views=batch_views)
    fg = FrameGather(len(cams), h, w, vr.device, group=group, dst=dst)
    fg.begin()
    if views:
        px, ld, st = vr.render([cams[i] for i in views])
        for j, view in enumerate(views):
            fg.send(view, px[j], ld[j], st[j])
    p, l, s = fg.finish()
    if p is None:
        return None, None, None
    return p.contiguous(), l, s

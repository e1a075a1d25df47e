"""Fused six-stage frame (sb/pipeline.py) on one B200.

``run_pipeline`` keeps the reference signature and returns the same
``PipelineResult``/``RenderStats``; stage times come from CUDA events recorded
between the kernels of one frame.  ``Rasterizer`` owns the persistent
workspace of a (scene size, resolution) and can capture a whole frame into a
CUDA graph — the serving/benchmark path, with no host synchronisation.

Stage → kernels (csrc/):
  preprocess    k_preprocess (fp64 projection + culling + touched counts)
  inclusivesum  compaction scan, depth-rank radix sort, pair-offset scan
  duplicate     k_emit (rank-ordered pairs + render records)
  sort          stable radix sort of pairs by tile id
  ranges        tile spans (+ export of reference-layout keys / indices)
  render        k_render (blend + load map + load-stat epilogue)
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

from . import _lib
from .metrics import LoadStats
from .projection import (ALPHA_LOW, COV_DILATION, CullingMode, Projection, as_device_scene,
                         scene_struct)
from .render import TERMINATION_THRESHOLD, Image, LoadMap
from .scene import DeviceScene
from .tiling import TileGrid, TilePairList

STAGE_NAMES = ("preprocess", "inclusivesum", "duplicate", "sort", "ranges", "render")

_TIME_QUANTUM = 2.0 ** -30  # seconds; makes the bucket identity exact in fp64


@dataclass(frozen=True)
class RenderStats:
    """Timings and counters of one frame (sb/pipeline.py:25-73)."""

    mode: CullingMode
    alpha_low: float
    gaussian_count: int
    culled_gaussians: int
    pair_count: int
    t_preprocess: float
    t_inclusivesum: float
    t_duplicate: float
    t_sort: float
    t_ranges: float
    t_render: float

    @property
    def e_g(self) -> float:
        return self.t_preprocess + self.t_inclusivesum + self.t_duplicate

    @property
    def e_n(self) -> float:
        return self.t_sort + self.t_ranges

    @property
    def e_p(self) -> float:
        return self.t_render

    @property
    def total_seconds(self) -> float:
        return (self.t_preprocess + self.t_inclusivesum + self.t_duplicate
                + self.t_sort + self.t_ranges + self.t_render)

    @property
    def fps(self) -> float:
        total = self.total_seconds
        return 1.0 / total if total > 0 else float("inf")

    def stage_seconds(self) -> dict:
        return {name: getattr(self, "t_" + name) for name in STAGE_NAMES}


@dataclass(eq=False)
class PipelineResult:
    """sb/pipeline.py:77-82, plus the epilogue's exact load statistics and
    two frame diagnostics: ``ambiguous_extents`` (culling extents whose ceil
    could change under a last-bit change of the fp64 log — 0 proves they
    equal numpy's, see csrc/adr_common.cuh:ceil_ambiguous) and
    ``nan_colors`` (valid Gaussians with a NaN colour channel)."""

    image: Image
    load_map: LoadMap
    stats: RenderStats
    projection: Projection
    pairs: TilePairList
    load_stats: LoadStats = None
    ambiguous_extents: int = 0
    nan_colors: int = 0


class StaleGraphError(RuntimeError):
    """A captured frame graph outlived the buffers it points at."""


class FrameGraph:
    """A CUDA graph of one frame, bound to its Rasterizer's buffer generation.

    Growing the pair capacity reallocates the buffers the graph's kernels
    point at; replaying a graph captured before that would touch freed
    memory, so ``replay`` refuses (``StaleGraphError``).  After a replay,
    ``Rasterizer.truncated()`` tells whether the frame needed more pairs than
    the capacity (its outputs are then incomplete)."""

    def __init__(self, graph, rast: "Rasterizer"):
        self.graph = graph
        self.rast = rast
        self.generation = rast.generation

    def replay(self) -> None:
        if self.generation != self.rast.generation:
            raise StaleGraphError("pair buffers were reallocated after capture; capture again")
        self.graph.replay()


def _estimate_capacity(n: int) -> int:
    return 16 * n + (1 << 16)


class Rasterizer:
    """Persistent workspace for frames of N Gaussians at W x H.

    Buffers (CUDA tensors): the Projection, image, load map, tile ranges, the
    sorted pair export (keys uint64, Gaussian indices int32), counters, load
    statistics and the library scratch, sized for ``pair_capacity`` pairs.
    """

    def __init__(self, width: int, height: int, n: int, device=None, pair_capacity: int = 0,
                 export_pairs: bool = True, timing: bool = True):
        import torch

        self.grid = TileGrid(width, height)
        self.width, self.height, self.n = int(width), int(height), int(n)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.export_pairs = export_pairs
        dev = self.device
        self.proj = Projection.empty(self.n, CullingMode.AABB, ALPHA_LOW, dev)
        self.pixels = torch.empty((self.height, self.width, 3), dtype=torch.float32, device=dev)
        self.load = torch.empty((self.height, self.width), dtype=torch.int32, device=dev)
        self.ranges = torch.empty((self.grid.n_tiles, 2), dtype=torch.int64, device=dev)
        self.counters = torch.zeros(8, dtype=torch.int64, device=dev)
        self.stats = torch.zeros(3, dtype=torch.int64, device=dev)  # adr_load_stats (24 B)
        self.cap = 0
        self.generation = 0   # bumped whenever the pair buffers are reallocated
        self.keys = self.gidx = self.scratch = None
        self._ensure_capacity(pair_capacity or _estimate_capacity(self.n))
        self.events = None
        self._ev_handles = None
        if timing:
            self.events = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
            with torch.cuda.device(dev):
                for e in self.events:
                    e.record()  # materialise the cudaEvent_t
            self._ev_handles = (ctypes.c_void_p * 7)(*[e.cuda_event for e in self.events])

    # -- buffers ------------------------------------------------------------
    def _ensure_capacity(self, cap: int) -> None:
        import torch

        cap = int(cap)
        if cap <= self.cap:
            return
        dev = self.device
        if self.export_pairs:
            self.keys = torch.empty(cap, dtype=torch.uint64, device=dev)
        # sorted Gaussian indices: the render's record index, always produced
        self.gidx = torch.empty(cap, dtype=torch.int32, device=dev)
        nbytes = _lib.lib().adr_frame_scratch_bytes(self.n, self.width, self.height, cap)
        self.scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.cap = cap
        self.generation += 1
        # the frame writes mean2d / conic / opacity / color only into its
        # 48-byte render record (adr_frame_buffers.projection_in_record): the
        # Projection's four fields are strided views of that record
        off = _lib.lib().adr_frame_record_offset(self.n, self.width, self.height, cap)
        rec = self.scratch[off: off + 48 * self.n].view(torch.float32).view(self.n, 12)
        self.proj.mean2d, self.proj.conic = rec[:, 0:2], rec[:, 2:5]
        self.proj.opacity, self.proj.color = rec[:, 5], rec[:, 6:9]

    def fit_capacity(self, pairs: int, slack: float = 1.02) -> None:
        """Size the pair buffers to `pairs` (+slack): grids of the pair-parallel
        kernels scale with the capacity, so a tight capacity is faster."""
        cap = int(pairs * slack) + 1024
        if cap != self.cap:
            self.cap = 0
            self._ensure_capacity(cap)

    def _buffers(self, timed: bool) -> _lib.FrameBuffers_t:
        b = _lib.FrameBuffers_t()
        b.proj = self.proj.struct(contiguous=False)
        b.d_pixels, b.d_load = _lib.ptr(self.pixels), _lib.ptr(self.load)
        b.d_keys = _lib.ptr(self.keys) if self.export_pairs else None
        b.d_gidx = _lib.ptr(self.gidx)
        b.d_ranges, b.d_counters = _lib.ptr(self.ranges), _lib.ptr(self.counters)
        b.d_stats, b.d_hist, b.hist_bins = _lib.ptr(self.stats), None, 0
        b.d_scratch, b.scratch_bytes = _lib.ptr(self.scratch), self.scratch.numel()
        b.pair_capacity = self.cap
        b.events = ctypes.cast(self._ev_handles, ctypes.c_void_p) if (timed and self._ev_handles) else None
        b.projection_in_record = 1
        return b

    # -- frames -------------------------------------------------------------
    def launch(self, scene: DeviceScene, cam, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
               dilation=COV_DILATION, term_threshold=TERMINATION_THRESHOLD, stream=None,
               timed: bool = False) -> None:
        """Enqueue one frame on `stream` (default: current); no host sync."""
        import torch

        mode = CullingMode(mode)
        if len(scene) != self.n:
            raise ValueError("scene size does not match the rasterizer")
        if (int(cam.width), int(cam.height)) != (self.width, self.height):
            raise ValueError("camera resolution does not match the rasterizer")
        self.proj.mode, self.proj.alpha_low = mode, alpha_low
        with torch.cuda.device(self.device):
            st = stream if stream is not None else torch.cuda.current_stream()
            _lib.check(_lib.lib().adr_render_frame(
                scene_struct(scene), _lib.camera_struct(cam), _lib.MODE_CODES[mode.value],
                float(alpha_low), float(dilation), float(term_threshold),
                ctypes.byref(self._buffers(timed)), _lib.stream_handle(st)))

    def _check_frame(self, scene: DeviceScene, cam) -> None:
        if len(scene) != self.n:
            raise ValueError("scene size does not match the rasterizer")
        if (int(cam.width), int(cam.height)) != (self.width, self.height):
            raise ValueError("camera resolution does not match the rasterizer")

    def launch_post(self, scene: DeviceScene, cam, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
                    dilation=COV_DILATION, term_threshold=TERMINATION_THRESHOLD, stream=None,
                    timed: bool = False) -> None:
        """Enqueue stages 2-6 of a frame whose stage 1 ran through
        ``preprocess_views`` into this rasterizer (same scene, camera, mode and
        alpha_low), on `stream` after that launch; no host sync."""
        import torch

        mode = CullingMode(mode)
        self._check_frame(scene, cam)
        self.proj.mode, self.proj.alpha_low = mode, alpha_low
        with torch.cuda.device(self.device):
            st = stream if stream is not None else torch.cuda.current_stream()
            _lib.check(_lib.lib().adr_render_frame_post(
                scene_struct(scene), _lib.camera_struct(cam), _lib.MODE_CODES[mode.value],
                float(alpha_low), float(dilation), float(term_threshold),
                ctypes.byref(self._buffers(timed)), _lib.stream_handle(st)))

    def pair_count(self) -> int:
        return int(self.counters[0].item())

    def truncated(self) -> bool:
        """True when the last frame needed more pairs than the capacity: its
        pair list, ranges and image are incomplete (counters[6]; syncs)."""
        return bool(self.counters[6].item())

    def render(self, scene, cam, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
               dilation=COV_DILATION, term_threshold=TERMINATION_THRESHOLD) -> PipelineResult:
        """One frame with stage timing; grows the pair buffers and re-runs when
        the frame needs more pairs than the current capacity."""
        import torch

        if not 0.0 < alpha_low < 1.0:
            raise ValueError("alpha_low must lie in (0, 1)")
        if dilation < 0:
            raise ValueError("dilation must be non-negative")
        mode = CullingMode(mode)
        ds = as_device_scene(scene, self.device)
        while True:
            self.launch(ds, cam, mode, alpha_low, dilation, term_threshold, timed=True)
            torch.cuda.synchronize(self.device)
            if not self.truncated():
                break
            self._ensure_capacity(int(self.pair_count() * 1.25) + 1024)
        return self.result(mode, alpha_low)

    def result(self, mode, alpha_low) -> PipelineResult:
        """Package the buffers of the last (synchronised) frame."""
        ctr = self.counters.cpu().tolist()
        p, culled = int(ctr[0]), int(ctr[1])
        t = [0.0] * 6
        if self.events is not None:
            for i in range(6):
                ms = self.events[i].elapsed_time(self.events[i + 1])
                t[i] = round(ms * 1e-3 / _TIME_QUANTUM) * _TIME_QUANTUM
        stats = RenderStats(mode=CullingMode(mode), alpha_low=alpha_low, gaussian_count=self.n,
                            culled_gaussians=culled, pair_count=p, t_preprocess=t[0],
                            t_inclusivesum=t[1], t_duplicate=t[2], t_sort=t[3], t_ranges=t[4],
                            t_render=t[5])
        s = self.stats.cpu().tolist()
        mn = s[2] & 0xFFFFFFFF
        mx = (s[2] >> 32) & 0xFFFFFFFF
        mn = mn - (1 << 32) if mn >= (1 << 31) else mn
        mx = mx - (1 << 32) if mx >= (1 << 31) else mx
        npx = self.width * self.height
        load_stats = LoadStats.from_moments(npx, int(s[0]), int(s[1]), mn, mx)
        keys = self.keys[:p] if self.export_pairs else None
        pairs = TilePairList(keys=keys, gaussian_indices=self.gidx[:p], tile_ranges=self.ranges)
        return PipelineResult(image=Image(self.width, self.height, self.pixels),
                              load_map=LoadMap(self.width, self.height, self.load), stats=stats,
                              projection=self.proj, pairs=pairs, load_stats=load_stats,
                              ambiguous_extents=int(ctr[5]), nan_colors=int(ctr[4]))

    def capture(self, scene: DeviceScene, cam, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
                dilation=COV_DILATION, term_threshold=TERMINATION_THRESHOLD):
        """Capture one whole frame into a ``FrameGraph`` (replay with ``g.replay()``).

        The capacity must already hold the frame's pairs (run ``render`` once);
        a replay whose frame outgrows it sets ``truncated()``."""
        import torch

        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.launch(scene, cam, mode, alpha_low, dilation, term_threshold, stream=s)  # warm
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(g, stream=s):
            self.launch(scene, cam, mode, alpha_low, dilation, term_threshold, stream=s)
        torch.cuda.synchronize(self.device)
        return FrameGraph(g, self)


MAX_BATCH_VIEWS = 8   # views per preprocess_views launch (adr_preprocess_views)


def preprocess_views(scene: DeviceScene, cams, rasts, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
                     dilation=COV_DILATION, stream=None) -> None:
    """Stage 1 of ``len(cams)`` (1..8) frames of one scene in ONE launch: each
    Gaussian and its SH coefficients are read once, its view-independent terms
    evaluated once, and view v's Projection / render record / tile rects /
    depth keys land in ``rasts[v]`` (one Rasterizer per view, distinct) —
    bit-identical to ``rasts[v].launch(scene, cams[v])``'s stage 1.  Follow
    with ``rasts[v].launch_post(scene, cams[v], ...)`` per view (any stream
    ordered after this one)."""
    import torch

    cams, rasts = list(cams), list(rasts)
    if not 1 <= len(cams) <= MAX_BATCH_VIEWS:
        raise ValueError(f"preprocess_views takes 1..{MAX_BATCH_VIEWS} views")
    if len(rasts) != len(cams):
        raise ValueError("one Rasterizer per view")
    if len({id(r) for r in rasts}) != len(rasts):
        raise ValueError("every view needs its own Rasterizer")
    mode = CullingMode(mode)
    for r, c in zip(rasts, cams):
        r._check_frame(scene, c)
        if r.device != rasts[0].device:
            raise ValueError("all rasterizers must live on one device")
        r.proj.mode, r.proj.alpha_low = mode, alpha_low
    cam_arr = (_lib.Camera_t * len(cams))(*[_lib.camera_struct(c) for c in cams])
    buf_arr = (_lib.FrameBuffers_t * len(rasts))(*[r._buffers(False) for r in rasts])
    with torch.cuda.device(rasts[0].device):
        st = stream if stream is not None else torch.cuda.current_stream()
        _lib.check(_lib.lib().adr_preprocess_views(
            scene_struct(scene), cam_arr, len(cams), _lib.MODE_CODES[mode.value], float(alpha_low),
            float(dilation), buf_arr, _lib.stream_handle(st)))


def render_views_batched(scene: DeviceScene, cams, rasts, mode=CullingMode.AABB, alpha_low=ALPHA_LOW,
                         dilation=COV_DILATION, term_threshold=TERMINATION_THRESHOLD, stream=None) -> None:
    """Enqueue whole frames of ``len(cams)`` (1..8) views of one scene on one
    stream: one ``preprocess_views`` launch, then each view's stages 2-6 in
    ``rasts[v]`` (read the results with ``rasts[v].result(...)`` after a
    sync).  Frames equal ``rasts[v].launch(scene, cams[v])`` bit for bit."""
    preprocess_views(scene, cams, rasts, mode, alpha_low, dilation, stream)
    for r, c in zip(rasts, cams):
        r.launch_post(scene, c, mode, alpha_low, dilation, term_threshold, stream=stream)


_workspace = threading.local()   # per host thread: {(device, N, W, H): Rasterizer}


def run_pipeline(scene, cam, mode: CullingMode = CullingMode.AABB, alpha_low: float = ALPHA_LOW,
                 threads: int = 1, dilation: float = COV_DILATION,
                 term_threshold: float = TERMINATION_THRESHOLD) -> PipelineResult:
    """All six stages for one scene/camera/mode (sb/pipeline.py:85-124).

    ``scene``: a DeviceScene (CUDA, or CPU — e.g. pinned — which is uploaded),
    a SceneArrays / reference Scene (uploaded as fp32 when every value is
    exactly representable, else fp64).  The frame's workspace (pair buffers,
    scratch) is kept per (device, N, W, H) and host thread and reused; the
    returned arrays are fresh CUDA tensors owned by the caller, with the
    reference's dtypes (gaussian_indices int64, keys uint64 bit patterns).
    ``threads`` is accepted for signature compatibility and never changes
    any output."""
    import torch

    mode = CullingMode(mode)
    grid = TileGrid(width=cam.width, height=cam.height)
    if not 0.0 < alpha_low < 1.0:
        raise ValueError("alpha_low must lie in (0, 1)")
    if dilation < 0:
        raise ValueError("dilation must be non-negative")
    ds = as_device_scene(scene)
    cache = getattr(_workspace, "rast", None)
    if cache is None:
        cache = _workspace.rast = {}
    key = (str(ds.device), len(ds), grid.width, grid.height)
    r = cache.get(key)
    if r is None:
        r = cache[key] = Rasterizer(grid.width, grid.height, len(ds), device=ds.device)
    res = r.render(ds, cam, mode, alpha_low, dilation, term_threshold)
    # hand the caller its own copies; the workspace stays with the cache
    p = res.stats.pair_count
    pairs = TilePairList(keys=r.keys[:p].clone() if r.export_pairs else None,
                         gaussian_indices=r.gidx[:p].to(torch.int64),
                         tile_ranges=r.ranges.clone())
    return PipelineResult(image=Image(r.width, r.height, r.pixels.clone()),
                          load_map=LoadMap(r.width, r.height, r.load.clone()),
                          stats=res.stats, projection=r.proj.clone(), pairs=pairs,
                          load_stats=res.load_stats, ambiguous_extents=res.ambiguous_extents,
                          nan_colors=res.nan_colors)

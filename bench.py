#!/usr/bin/env python
"""Benchmark: rendered frames/s and Gaussian-tile pairs/frame (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W] [--config garden] [--views V] [--impl ours|reference]

One step = one batch of V camera views rendered through all six stages
(sb/pipeline.py:85-124), view-sharded over the ranks (rank r
renders the contiguous slice shard_views(V, N, r)), with every frame + its
stats gathered to rank 0 over NCCL point-to-point transfers that overlap the
rendering — the gather is inside the timed region.  Rank 0 prints ONE JSON
line; value = V x K / (max over ranks of the CUDA-event time of K steps).

Batch size: V = 8 x N for the single-view configurations (garden = BASELINE
configs[2], the headline; truck; config1) — weak scaling, 8 views per GPU;
V = 64 for playroom (configs[3]) and 256 for stress (configs[4]) at every N —
strong scaling, as BASELINE states them.  Synthetic scene (seeded
generate_synthetic draws + SH rest N(0, 0.3^2), values rounded to fp32),
spec scale U(0.004, 0.016), anisotropy U(1, 4), opacity U(0.01, 0.6), orbit
cameras at radius 2.6, fov 60; rank 0 builds it and broadcasts it.  Inputs
(scene >= 0.5 GB, pair buffers) are larger than the 126 MB L2, so no
explicit L2 flush is needed.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BIG_SPEC = dict(extent=1.0, scale_range=(0.004, 0.016), anisotropy_range=(1.0, 4.0),
                opacity_range=(0.01, 0.6))
CONFIGS = {
    # BASELINE.json configs[0]: the reference's own test workload
    "config1": dict(n=10_000, w=256, h=256, mode="aabb", sh=3, spec={}, radius=5.0,
                    name="synthetic 10k-Gaussian scene, 1 view 256x256, SH3 (configs[0])"),
    # configs[1]: Tanks&Temples-Truck scale, adaptive radius only
    "truck": dict(n=2_500_000, w=979, h=546, mode="circle", sh=3, spec=BIG_SPEC, radius=2.6,
                  name="synthetic T&T-Truck scale: 2.5M Gaussians 979x546, adaptive radius (configs[1])"),
    # configs[2]: Mip-NeRF360-garden scale, AABB + load map/stats — the north_star target
    "garden": dict(n=5_800_000, w=1297, h=840, mode="aabb", sh=3, spec=BIG_SPEC, radius=2.6,
                   name="synthetic Mip-NeRF360-garden scale: 5.8M Gaussians 1297x840, "
                        "adaptive radius + AABB + load map (configs[2])"),
    # configs[3]: Deep-Blending-playroom scale, view batch
    "playroom": dict(n=2_300_000, w=1264, h=832, mode="aabb", sh=3, spec=BIG_SPEC, radius=2.6,
                     name="synthetic DB-playroom scale: 2.3M Gaussians 1264x832 (configs[3])"),
    # configs[4]: stress
    "stress": dict(n=10_000_000, w=1920, h=1080, mode="aabb", sh=3, spec=BIG_SPEC, radius=2.6,
                   name="stress: 10M Gaussians 1920x1080 (configs[4])"),
}
VIEWS_PER_RANK = 8
# fixed view batches of the multi-view configurations (strong scaling)
FIXED_VIEWS = {"playroom": 64, "stress": 256}
METRIC = "rendered frames/sec and Gaussian-tile pairs/frame; 1/2/4/8 B200 view-sharded"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="garden")
    ap.add_argument("--views", type=int, default=0,
                    help="views per step (default: 8 per GPU; playroom 64, stress 256)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of sampled CPU render")
    ap.add_argument("--streams", type=int, default=8,
                    help="views in flight per GPU: one Rasterizer + stream each (frames of different "
                         "views overlap; each frame is still one CUDA graph)")
    ap.add_argument("--batch-views", type=int, default=-1,
                    help="views per stage-1 launch (adr_preprocess_views: the scene is read once for the "
                         "batch); 1 = one adr_render_frame graph per view; -1 (default): 8 for scenes of "
                         ">= 262144 Gaussians, else 1 (a 10k-Gaussian frame is launch-bound: notes.md "
                         "experiment 21)")
    ap.add_argument("--slot-sets", type=int, default=0,
                    help="batched stage 1: slot sets the groups alternate over (2: a group's stage 1 "
                         "overlaps the previous group's frames, also across steps); 0 (default): 2 when "
                         "a step has several groups, else 1 (garden: 1 set 832-837 vs 2 sets 822-829 "
                         "frames/s; truck the other way round, 1933 vs 1967: notes.md experiment 22)")
    ap.add_argument("--e2e-streams", type=int, default=4,
                    help="views in flight in the e2e legs (single-view C-ABI frame calls; notes.md "
                         "experiments 14 and 21)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def scene_arrays(cfg):
    from paper_2409_08669_b200 import SyntheticSpec, synthetic_arrays

    return synthetic_arrays(2409, cfg["n"], SyntheticSpec(**cfg["spec"]), sh_degree=cfg["sh"],
                            float32=True)


def cameras(cfg, n_views):
    from paper_2409_08669_b200.views import orbit_cameras

    return orbit_cameras(n_views, cfg["w"], cfg["h"], radius=cfg["radius"],
                         background=(0.0, 0.0, 0.0))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler (B200_PROFILING.md clocks line) over the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
                for i, nm in enumerate(names):
                    if r[5 + i].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def frame_algorithmic_bytes(n, k_sh, pairs, w, h):
    """B_alg = N(112 + 12K) + 84 P + 16 HW."""
    return n * (112 + 12 * k_sh) + 84 * pairs + 16 * w * h


def render_kernel_bytes(pairs, w, h, n_tiles):
    """Algorithmic bytes of one k_render launch: per pair the 4 B rank plus the
    48 B record gathered into shared memory, per tile its 16 B span, per pixel
    12 B RGB + 4 B load written."""
    return 52 * pairs + 16 * n_tiles + 16 * w * h


def cpu_reference_sample(cfg, arrays, cam, budget_s, threads):
    """The oracle port (C, OpenMP) on a bounded sample of one frame: the full
    preprocess/count/scan/duplicate/sort/ranges plus every s-th tile of the
    render, extrapolated to the full tile count."""
    from oracle import oracle as orc

    tx, ty = orc.grid_dims(cfg["w"], cfg["h"])
    nt = tx * ty
    scene = dict(centers=arrays.centers, scales=arrays.scales, rotations=arrays.rotations,
                 opacities=arrays.opacities, sh=arrays.sh, sh_degree=cfg["sh"])
    t0 = time.perf_counter()
    proj = orc.preprocess(scene, cam, cfg["mode"], threads=threads)
    t1 = time.perf_counter()
    counts = orc.touched_counts(proj, cfg["w"], cfg["h"])
    offs = orc.inclusive_sum(counts)
    t2 = time.perf_counter()
    keys, gidx = orc.duplicate_with_keys(proj, offs, cfg["w"], cfg["h"])
    t3 = time.perf_counter()
    sk, sg = orc.sort_pairs(keys, gidx)
    t4 = time.perf_counter()
    ranges = orc.identify_tile_ranges(sk, nt)
    t5 = time.perf_counter()
    # calibrate the render sample: one probe stride, then size to the budget
    stride = max(1, nt // 64)
    tp = time.perf_counter()
    orc.render(proj, sg, ranges, cam, threads=threads, tile_stride=stride)
    probe = time.perf_counter() - tp
    probe_tiles = len(range(0, nt, stride))
    per_tile = probe / probe_tiles
    want = max(probe_tiles, min(nt, int(budget_s / max(per_tile, 1e-9))))
    stride = max(1, nt // want)
    tr = time.perf_counter()
    orc.render(proj, sg, ranges, cam, threads=threads, tile_stride=stride, tile_phase=1 % stride)
    t_render_sample = time.perf_counter() - tr
    sampled = len(range(1 % stride, nt, stride))
    t_render = t_render_sample * nt / sampled
    total = (t1 - t0) + (t2 - t1) + (t3 - t2) + (t4 - t3) + (t5 - t4) + t_render
    return {"fps": 1.0 / total, "frame_s": total, "pairs": int(len(sk)),
            "stages_s": {"preprocess": t1 - t0, "inclusivesum": t2 - t1, "duplicate": t3 - t2,
                         "sort": t4 - t3, "ranges": t5 - t4, "render": t_render},
            "sample": f"1 frame of {cfg['n']} Gaussians at {cfg['w']}x{cfg['h']}: full stages 1-5, "
                      f"render of {sampled}/{nt} tiles (every {stride}-th) extrapolated to all tiles"}


def batch_views(args, cfg_name, world):
    if args.views:
        return args.views, "strong"
    if cfg_name in FIXED_VIEWS:
        return FIXED_VIEWS[cfg_name], "strong"
    return VIEWS_PER_RANK * world, "weak"


def config_dict(cfg, args, views, world, pairs, scaling):
    return {"workload": cfg["name"], "gaussians": cfg["n"], "width": cfg["w"], "height": cfg["h"],
            "mode": cfg["mode"], "sh_degree": cfg["sh"], "pairs_per_frame": pairs,
            "views_per_step": views, "scaling": scaling,
            "parallelism": f"view-sharded x{world}",
            "l2": "inputs larger than L2 (scene %.2f GB)" % (cfg["n"] * (44 + 12 * (cfg["sh"] + 1) ** 2) / 1e9)}


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference algorithm on the host cores (the C
    oracle port, OpenMP, every host thread; the reference itself is pure numpy
    at ~90 s per 5.8M frame).  Same configuration, cameras and metric as our
    arm: step s renders view s mod V of the same orbit (full stages 1-5 and a
    tile-strided render sample extrapolated to all tiles)."""
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.lib()
    threads = os.cpu_count() or 1
    arrays = scene_arrays(cfg)
    views, scaling = batch_views(args, args.config, world)
    cams = cameras(cfg, views)
    budget = max(2.0, min(args.cpu_budget, 20.0)) / 3.0
    for s in range(max(0, min(args.warmup, 1))):
        cpu_reference_sample(cfg, arrays, cams[s % views], budget / 2, threads)
    steps = max(1, min(args.steps, 20))
    samples = [cpu_reference_sample(cfg, arrays, cams[s % views], budget, threads) for s in range(steps)]
    frame_s = sum(x["frame_s"] for x in samples) / len(samples)
    fps = 1.0 / frame_s
    pairs = float(np.mean([x["pairs"] for x in samples]))
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": frame_s * 1e3,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64+f32",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, args, views, world, pairs, scaling),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": f"{steps} frames, view s mod {views} of the orbit; each: " + samples[0]["sample"]},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "stages_s": samples[0]["stages_s"]}
    print(json.dumps(line), flush=True)


def run_ours(args, cfg, rank, world, local):
    import torch

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import _lib
    from paper_2409_08669_b200.views import FrameGather, broadcast_scene, shard_views

    # one rank per GPU over NCCL; ADR_BENCH_BACKEND=gloo is a functional test of
    # the multi-rank path on a one-GPU box (ranks share device 0; gloo moves
    # the frames through host memory), never a measurement
    backend = os.environ.get("ADR_BENCH_BACKEND", "nccl")
    gpu = local if backend == "nccl" else local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def reduce_(t, op=None):
        """all_reduce on the device over NCCL, through host memory over gloo."""
        if backend == "nccl":
            dist.all_reduce(t, op=op or dist.ReduceOp.SUM)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=op or dist.ReduceOp.SUM)
        t.copy_(h)
        return t
    L = _lib.lib()
    t_setup = time.perf_counter()
    # scene: built once on rank 0, broadcast to the others
    arrays, host, ds = None, None, None
    if rank == 0:
        arrays = scene_arrays(cfg)
        host = ab.DeviceScene.from_arrays(arrays, cfg["sh"], "cpu", torch.float32).pin_memory()
        ds = host.to(dev)
    if world > 1:
        ds = broadcast_scene(ds, cfg["n"], cfg["sh"], dev)
        if rank != 0:
            host = ds.to("cpu").pin_memory()   # this rank's host copy for the e2e legs
    views, scaling = batch_views(args, args.config, world)
    cams = cameras(cfg, views)
    mine = list(shard_views(views, world, rank))
    n_mine = len(mine)
    rast = ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"], device=dev)
    pairs, stage_ms = [], []
    for v in mine:   # size the pair buffers for every view of this rank
        res = rast.render(ds, cams[v], mode=cfg["mode"])
        pairs.append(res.stats.pair_count)
    rast.fit_capacity(max(pairs) if pairs else 0)
    v0 = mine[0] if mine else 0
    for _ in range(10):   # per-stage CUDA-event durations (the roofline's denominators)
        res = rast.render(ds, cams[v0], mode=cfg["mode"])
        stage_ms.append({k: v * 1e3 for k, v in res.stats.stage_seconds().items()})
    first = rast.render(ds, cams[v0], mode=cfg["mode"])
    load_stats = first.load_stats
    culled = first.stats.culled_gaussians
    before = L.adr_kernel_launches()
    rast.launch(ds, cams[v0], mode=cfg["mode"])
    torch.cuda.synchronize(dev)
    launches_per_frame = L.adr_kernel_launches() - before
    # views in flight: view j of this rank renders through slot j % K on its own stream
    n_fly = max(1, min(args.streams, max(n_mine, 1)))
    n_e2e = max(1, min(args.e2e_streams, n_fly))   # views in flight in the e2e legs
    rasts = [rast] + [ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"], device=dev, pair_capacity=rast.cap,
                                    timing=False) for _ in range(n_fly - 1)]
    streams = [torch.cuda.Stream(dev) for _ in range(n_fly)]
    graphs = [rasts[j % n_fly].capture(ds, cams[v], mode=cfg["mode"]) for j, v in enumerate(mine)]
    # batched stage 1: groups of G consecutive views share one preprocess_views
    # launch (one scene read); two slot sets alternate so group g+1's stage 1
    # overlaps group g's binning + render
    bv = args.batch_views if args.batch_views > 0 else (ab.MAX_BATCH_VIEWS if cfg["n"] >= 262144 else 1)
    G = max(1, min(bv, ab.MAX_BATCH_VIEWS, max(n_mine, 1)))
    groups = [list(range(i, min(i + G, n_mine))) for i in range(0, n_mine, G)] if G > 1 else []
    # two slot sets: consecutive groups (also across steps) alternate, so the
    # next group's stage 1 overlaps the previous group's binning + render
    n_sets = (max(1, min(2, args.slot_sets)) if args.slot_sets > 0 else min(2, len(groups))) if groups else 0
    slots, pre_graphs, post_graphs, pre_streams = [], [], [], []
    if groups:
        slots = rasts[:G * n_sets] + [ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"], device=dev, pair_capacity=rast.cap,
                                                    timing=False) for _ in range(G * n_sets - len(rasts))]
        pre_streams = [torch.cuda.Stream(dev) for _ in range(n_sets)]

        def capture(fn):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(torch.cuda.current_stream(dev))
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(g, stream=cs):
                fn(cs)
            torch.cuda.synchronize(dev)
            return g

        # pre_graphs[set][group], post_graphs[set][view j of this rank]
        pre_graphs = [[None] * len(groups) for _ in range(n_sets)]
        post_graphs = [[None] * n_mine for _ in range(n_sets)]
        for ss in range(n_sets):
            for gi, grp in enumerate(groups):
                sl = [slots[ss * G + q] for q in range(len(grp))]
                gc = [cams[mine[j]] for j in grp]
                before_b = L.adr_kernel_launches()
                ab.render_views_batched(ds, gc, sl, mode=cfg["mode"])   # eager run before capture
                torch.cuda.synchronize(dev)
                if gi == 0 and ss == 0:
                    launches_per_frame = (L.adr_kernel_launches() - before_b) / len(grp)
                for r_ in sl:
                    assert not r_.truncated()
                pre_graphs[ss][gi] = capture(lambda cs, gc=gc, sl=sl: ab.preprocess_views(
                    ds, gc, sl, mode=cfg["mode"], stream=cs))
                for q, j in enumerate(grp):
                    post_graphs[ss][j] = capture(lambda cs, r_=sl[q], c_=gc[q]: r_.launch_post(
                        ds, c_, mode=cfg["mode"], stream=cs))
    fg = FrameGather(views, cfg["h"], cfg["w"], dev) if world > 1 else None
    zero = torch.zeros(1, dtype=torch.int64, device=dev)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(dev)

    def step(gather: bool, join: bool = True):
        """One batch: this rank's views (frames of different views overlap on
        the slot streams); with `gather`, each frame is shipped to rank 0 as
        soon as it is rendered and the step ends when every transfer landed."""
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        for st in streams:
            st.wait_event(ev0)
        if fg is not None and gather:
            fg.begin()
        for j, v in enumerate(mine):
            k = j % n_fly
            with torch.cuda.stream(streams[k]):
                graphs[j].replay()
                if fg is not None and gather:
                    r = rasts[k]
                    fg.send(v, r.pixels, r.load, torch.cat([r.counters[0:2], r.stats[0:3], zero]))
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)
        if fg is not None and gather:
            fg.finish()

    bpre_ms = None
    if groups:   # the batched stage-1 launch alone (its roofline denominator)
        ts = []
        for _ in range(7):
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record(stream)
            pre_graphs[0][0].replay()
            q1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(q0.elapsed_time(q1))
        bpre_ms = statistics.median(ts[2:])

    gcount = [0]                                # groups issued so far (slot-set alternation)
    pending = [[] for _ in range(n_sets)]       # per slot set: events of its last group's frames

    def step_batched(gather: bool, join: bool = True):
        """One batch through batched stage 1: per group of G views one
        preprocess_views graph on its slot set's stream (waiting only for that
        set's previous frames), then each view's stages 2-6 graph on the
        in-flight streams (gathered like `step`).  Without `join` the next
        step's stage 1 may start while this step's last frames still run."""
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        for st in streams + pre_streams:
            st.wait_event(ev0)
        if fg is not None and gather:
            fg.begin()
        for gi, grp in enumerate(groups):
            ss = gcount[0] % n_sets
            gcount[0] += 1
            ps = pre_streams[ss]
            for e in pending[ss]:
                ps.wait_event(e)
            with torch.cuda.stream(ps):
                pre_graphs[ss][gi].replay()
            pe = torch.cuda.Event()
            pe.record(ps)
            used = []
            for q, j in enumerate(grp):
                k = j % n_fly
                streams[k].wait_event(pe)
                with torch.cuda.stream(streams[k]):
                    post_graphs[ss][j].replay()
                    if fg is not None and gather:
                        r = slots[ss * G + q]
                        fg.send(mine[j], r.pixels, r.load, torch.cat([r.counters[0:2], r.stats[0:3], zero]))
                if k not in used:
                    used.append(k)
            pending[ss] = []
            for k in used:
                e = torch.cuda.Event()
                e.record(streams[k])
                pending[ss].append(e)
        if join or (fg is not None and gather):
            for st in streams + pre_streams:
                ev = torch.cuda.Event()
                ev.record(st)
                stream.wait_event(ev)
        if fg is not None and gather:
            fg.finish()

    if groups:
        step = step_batched  # noqa: F811

    def timed(k_steps: int, gather: bool) -> float:
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k_steps):   # consecutive steps may overlap; the last one joins every stream
            step(gather, join=(i == k_steps - 1))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            reduce_(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        step(True)
    torch.cuda.synchronize(dev)
    # render-only (no gather): the per-rank rendering rate
    ms_render = timed(args.steps, gather=False)
    clocks = Clocks(gpu)
    clocks.start()
    time.sleep(0.3)
    ms = timed(args.steps, gather=True)   # the headline: render + gather to rank 0
    # keep the clock sampler under load >= 1.5 s; the step count derives from
    # the max-reduced time, so every rank runs the same number of gathered
    # steps (a wall-clock loop could leave one rank's frame sends unmatched)
    n_soak = int(math.ceil(max(0.0, 1.5 - ms * 1e-3) / max(ms * 1e-3 / args.steps, 1e-6)))
    for _ in range(n_soak):
        step(True)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    frames = views * args.steps
    value = frames / (ms * 1e-3)
    ms_per_step = ms / args.steps
    p_mean = float(np.mean(pairs)) if pairs else 0.0
    if dist:
        t = torch.tensor([p_mean * n_mine, float(n_mine)], dtype=torch.float64, device=dev)
        reduce_(t)
        p_mean = float(t[0] / max(t[1], 1.0))
    med = {k: statistics.median(d[k] for d in stage_ms) for k in stage_ms[0]}
    hbm, peak_kind = peaks()
    nt = rast.grid.n_tiles
    k_sh = (cfg["sh"] + 1) ** 2
    n = cfg["n"]
    # per-kernel evidence from the committed ncu summaries (profiles/ncu_summary.json)
    prof = ROOT / "profiles" / "ncu_summary.json"
    ncu = {}
    if prof.exists():
        try:
            ncu = json.loads(prof.read_text()).get(args.config, {})
        except Exception:
            ncu = {}
    # K1 (preprocess), HBM-bound: SURVEY.md §8(d) bytes = N(44 + 12K) scene read + 52 N Projection
    # write; the implementation also writes the 48 B render record + 8 B tile rect + 4 B depth key
    pre_bytes = n * (44 + 12 * k_sh) + n * 52
    pre_impl_bytes = n * (44 + 12 * k_sh) + n * (65 + 4) + (n - culled) * (48 + 8)
    pre_gbs = pre_bytes / (med["preprocess"] * 1e-3) / 1e9
    # binning (depth sort + supertile placement), §8(d): N·16 dup read + P·12 pair write + P·24 ideal sort pass
    bin_ms = med["inclusivesum"] + med["duplicate"] + med["sort"] + med["ranges"]
    bin_bytes = n * 16 + p_mean * 36
    rbytes = render_kernel_bytes(p_mean, cfg["w"], cfg["h"], nt)
    falg = frame_algorithmic_bytes(n, k_sh, p_mean, cfg["w"], cfg["h"])

    # e2e legs (per rank; aggregated over ranks)
    e2e = e2e_frame = e2e_res = e2e_rp = None
    # the e2e legs hold barriers and reductions: every rank must agree to run them
    run_e2e = not args.no_e2e and n_mine > 0
    if dist:
        t = torch.tensor([1.0 if run_e2e else 0.0], dtype=torch.float64, device=dev)
        reduce_(t, op=dist.ReduceOp.MIN)
        run_e2e = bool(t.item() > 0.5)
    if run_e2e:
        src = [host.centers, host.scales, host.rotations, host.opacities, host.sh]
        dst = [ds.centers, ds.scales, ds.rotations, ds.opacities, ds.sh]
        h2d = host.nbytes()
        slot_h = [(torch.empty_like(r.pixels, device="cpu").pin_memory(),
                   torch.empty_like(r.load, device="cpu").pin_memory()) for r in rasts]
        d2h_frame = slot_h[0][0].numel() * 4 + slot_h[0][1].numel() * 4
        k_e2e = max(3, min(args.steps, 10))
        # two device copies of the scene: step s+1's H2D copy (copy stream)
        # overlaps step s's frames; every step still moves its own scene in
        dst2 = [t.clone() for t in dst]
        ds2 = ab.DeviceScene(*dst2, sh_degree=ds.sh_degree)
        scenes, bufs = (ds, ds2), (dst, dst2)
        cstream = torch.cuda.Stream(dev)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        free = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_run(steps: int, views_per_step: int) -> float:
            """Per step: the scene H2D from pinned host memory, `views_per_step`
            of this rank's views through the C-ABI frame call (Rasterizer.launch,
            no graph) on the in-flight slots, each frame's image + load map D2H
            to pinned host memory."""
            torch.cuda.synchronize(dev)
            if dist:
                dist.barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            cstream.wait_event(a0)
            j = 0
            for s_ in range(steps):
                bb = s_ % 2
                with torch.cuda.stream(cstream):
                    if s_ >= 2:
                        cstream.wait_event(free[bb])
                    for x_, y_ in zip(bufs[bb], src):
                        x_.copy_(y_, non_blocking=True)
                    ready[bb].record(cstream)
                for st in streams:
                    st.wait_event(ready[bb])
                for _ in range(views_per_step):
                    k = j % n_e2e
                    rasts[k].launch(scenes[bb], cams[mine[j % n_mine]], mode=cfg["mode"], stream=streams[k])
                    with torch.cuda.stream(streams[k]):
                        slot_h[k][0].copy_(rasts[k].pixels, non_blocking=True)
                        slot_h[k][1].copy_(rasts[k].load, non_blocking=True)
                    j += 1
                for st in streams:
                    ev = torch.cuda.Event()
                    ev.record(st)
                    stream.wait_event(ev)
                free[bb].record(stream)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            return a0.elapsed_time(a1)

        e2e_run(2, n_mine)   # warm-up
        ems = e2e_run(k_e2e, n_mine)          # the bench's step: this rank's V/R views per scene upload
        fms = e2e_run(k_e2e, 1)               # one frame per scene upload
        # resident scene (serving): per step a new camera through the C-ABI
        # frame call on one of the in-flight slots, image+load map back
        torch.cuda.synchronize(dev)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for st in streams:
            st.wait_event(b0)
        n_res = max(args.steps, 8)
        for s_ in range(n_res):
            k = s_ % n_e2e
            rasts[k].launch(ds, cams[mine[s_ % n_mine]], mode=cfg["mode"], stream=streams[k])
            with torch.cuda.stream(streams[k]):
                slot_h[k][0].copy_(rasts[k].pixels, non_blocking=True)
                slot_h[k][1].copy_(rasts[k].load, non_blocking=True)
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)
        b1.record(stream)
        torch.cuda.synchronize(dev)
        rms = b0.elapsed_time(b1)
        # the literal drop-in call: run_pipeline(pinned host scene, camera) ->
        # PipelineResult; synchronous, wall clock per call
        ab.run_pipeline(host, cams[mine[0]], mode=cfg["mode"])
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        k_rp = max(2, min(args.steps, 6))
        w0 = time.perf_counter()
        for s_ in range(k_rp):
            res = ab.run_pipeline(host, cams[mine[s_ % n_mine]], mode=cfg["mode"])
            _ = res.image.pixels.cpu()
        rp_s = time.perf_counter() - w0
        if dist:
            t = torch.tensor([ems, fms, rms, rp_s], dtype=torch.float64, device=dev)
            reduce_(t, op=dist.ReduceOp.MAX)
            ems, fms, rms, rp_s = (float(v) for v in t.tolist())
        e2e = {"value": views * k_e2e / (ems * 1e-3), "unit": "frames/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h_frame * n_mine,
               # per rank: the scene upload is the bound (PCIe Gen5 x16 moves ~55 GB/s)
               "h2d_gbs_per_rank": h2d * k_e2e / (ems * 1e-3) / 1e9,
               "path": "per step (as in value: this rank's views of the batch): the scene H2D from pinned "
                       "host memory, every view through the C-ABI frame call (Rasterizer.launch, no graph), "
                       "each image + load map D2H to pinned host memory; double-buffered device scene (step "
                       "s+1's upload overlaps step s's frames)"}
        e2e_frame = {"value": world * k_e2e / (fms * 1e-3), "unit": "frames/s",
                     "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h_frame,
                     "path": "the same with one view per scene upload (run_pipeline semantics: every frame "
                             "re-sends its scene)"}
        e2e_res = {"value": world * n_res / (rms * 1e-3), "unit": "frames/s",
                   "h2d_bytes_per_step": ctypes.sizeof(_lib.Camera_t), "d2h_bytes_per_step": d2h_frame,
                   "path": "resident scene; per step Rasterizer.launch with a new camera (C-ABI call, "
                           "no graph) on one of the in-flight slots, image+load map copied to pinned host"}
        e2e_rp = {"value": world * k_rp / rp_s, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                  "d2h_bytes_per_step": slot_h[0][0].numel() * 4,
                  "path": "paper_2409_08669_b200.run_pipeline(pinned host DeviceScene, camera) per frame, "
                          "synchronous, wall clock (includes the scene upload, stage events, result copies)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        c = cpu_reference_sample(cfg, arrays, cams[0], args.cpu_budget, threads)
        cpu = {"value": c["fps"], "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": c["sample"], "stages_s": c["stages_s"]}

    if rank == 0:
        cfgd = config_dict(cfg, args, views, world, p_mean, scaling)
        cfgd.update({"step": f"{views} views rendered (view-sharded) + gathered to rank 0",
                     "frame": (f"stage 1 of {G} views per launch (preprocess_views graph, scene read once per "
                               f"group), stages 2-6 a CUDA graph per view, no host sync" if groups else
                               "CUDA graph per view, no host sync"),
                     "views_in_flight": n_fly, "e2e_views_in_flight": n_e2e,
                     "batch_views": G if groups else 1})
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64 preprocess / f32 blend (bit-exact)", "data": "synthetic",
            "config": cfgd,
            "pairs_per_frame": p_mean,
            "stages_ms": {"preprocess": med["preprocess"], "depth_sort": med["inclusivesum"],
                          "supertile_items": med["duplicate"], "pair_placement": med["sort"],
                          "render": med["render"]},
            "per_rank_fps_render_only": n_mine * args.steps / (ms_render * 1e-3),
            "render_only_value": views * args.steps / (ms_render * 1e-3),
            "gather": ("point-to-point to rank 0 (NCCL), overlapped with rendering, inside the timed region"
                       if world > 1 else "none (one rank)"),
            "sort_rates": {"depth_sort_keys_per_s": n / (med["inclusivesum"] * 1e-3),
                           "pair_binning_pairs_per_s": p_mean / ((med["duplicate"] + med["sort"]) * 1e-3)},
            "load_stats": {"mean": load_stats.mean, "std": load_stats.std, "min": load_stats.min,
                           "max": load_stats.max},
            # the dominant HBM-bound kernel: K1, the fp64 preprocess
            "roofline": {"bound": "hbm", "kernel": "k_preprocess", "achieved": pre_gbs, "peak": hbm,
                         "unit": "GB/s", "frac": pre_gbs / hbm,
                         "traffic": ncu.get("k_preprocess_dram_bytes"),
                         "bytes_per_launch": pre_bytes,
                         "bytes_rule": "SURVEY.md §8(d): N(44+12K) read + 52N write",
                         "impl_bytes_per_launch": pre_impl_bytes,
                         "impl_frac": pre_impl_bytes / (med["preprocess"] * 1e-3) / 1e9 / hbm,
                         "peak_kind": peak_kind,
                         "duration_ms": med["preprocess"],
                         "duration_source": "median of CUDA events around the stage in 10 frames of the "
                                            "bench view rendered one at a time (no other frame in flight)"},
            "batch_preprocess": None if bpre_ms is None else {
                "kernel": "k_preprocess_views", "views_per_launch": len(groups[0]), "ms": bpre_ms,
                "ms_per_view": bpre_ms / len(groups[0]),
                "bytes_per_launch": n * (44 + 12 * k_sh) + len(groups[0]) * n * 52,
                "bytes_rule": "SURVEY.md §8(d) with the scene read once per launch: N(44+12K) + views·52N",
                "achieved": (n * (44 + 12 * k_sh) + len(groups[0]) * n * 52) / (bpre_ms * 1e-3) / 1e9,
                "frac": (n * (44 + 12 * k_sh) + len(groups[0]) * n * 52) / (bpre_ms * 1e-3) / 1e9 / hbm,
                "duration_source": "median of CUDA events around the group-0 stage-1 graph replayed alone",
                "bound": "fp64-issue",
                "traffic": ncu.get("k_preprocess_views_dram_bytes"),
                "issue_active": ncu.get("k_preprocess_views_issue_active"),
                "fp64_pipe_active": ncu.get("k_preprocess_views_fp64_pipe")},
            "binning_roofline": {"bound": "hbm", "kernels": "depth sort + supertile items + pair placement",
                                 "bytes_per_frame": bin_bytes,
                                 "bytes_rule": "SURVEY.md §8(d): N·16 dup read + P·12 pair write + P·24 one ideal sort pass",
                                 "achieved": bin_bytes / (bin_ms * 1e-3) / 1e9, "peak": hbm,
                                 "frac": bin_bytes / (bin_ms * 1e-3) / 1e9 / hbm, "ms": bin_ms},
            "render_kernel": {"bound": "fp32-issue", "kernel": "k_render",
                              "gather_gbs": rbytes / (med["render"] * 1e-3) / 1e9, "bytes_per_launch": rbytes,
                              "traffic": ncu.get("k_render_dram_bytes"),
                              "fma_pipe_active": ncu.get("k_render_fma_pipe"),
                              "issue_active": ncu.get("k_render_issue_active"),
                              "warp_inst_per_s": ncu.get("k_render_warp_inst_per_s"),
                              "warp_inst_peak_per_s": 148 * 4 * (clk.get("sm_mhz") or 1965.0) * 1e6,
                              "note": "52 B/pair record gathers + outputs, served from L2; the limiter is FP32 "
                                      "issue for the exact numpy exp (FFMA2 + MUFU) and dependency latency"},
            "frame_roofline": {"bytes_per_frame": falg, "achieved_gbs": falg * value / world / 1e9,
                               "frac": falg * value / world / 1e9 / hbm,
                               "bytes_rule": "SURVEY.md §8(d): N(112+12K) + 84P + 16HW"},
            "clocks": clk, "gpu_launches": int(round(launches_per_frame * frames)),
            "launches_per_frame": launches_per_frame, "setup_s": setup_s,
        }
        if e2e:
            line["e2e"] = e2e
            line["e2e_frame_upload"] = e2e_frame
            line["e2e_resident"] = e2e_res
            line["e2e_run_pipeline"] = e2e_rp
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    run_ours(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()

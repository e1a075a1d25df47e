"""GPU: the view-sharded multi-GPU entry point with two real processes.

This run has one B200, and NCCL refuses two ranks on one GPU, so the two
ranks use the gloo backend (frames and the scene broadcast travel through
host memory) while both render on cuda:0 with the same kernels as the NCCL
path.  Rank 0 loads the scene and broadcasts it (``broadcast_scene``); each
rank renders its contiguous view slice (``render_views_sharded``); the frames
are gathered to rank 0 (``FrameGather``, point-to-point, view order) and must
equal single-process ``run_pipeline`` frames bit for bit."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu

N, W, H, V = 30000, 160, 120, 5


def _scene_arrays():
    import paper_2409_08669_b200 as ab

    spec = ab.SyntheticSpec(extent=1.0, scale_range=(0.004, 0.03), anisotropy_range=(1, 4),
                            opacity_range=(0.01, 0.9))
    return ab.synthetic_arrays(31, N, spec, sh_degree=3, float32=True)


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200.views import broadcast_scene, orbit_cameras, render_views_sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        src = None
        if rank == 0:
            src = ab.DeviceScene.from_arrays(_scene_arrays(), 3, "cuda:0", torch.float32)
        ds = broadcast_scene(src, N, 3, "cuda:0")
        cams = orbit_cameras(V, W, H, radius=2.6)
        px, ld, st = render_views_sharded(ds, cams, in_flight=2)
        if rank == 0:
            q.put((px.cpu().numpy().copy(), ld.cpu().numpy().copy(), st.cpu().numpy().copy()))
        else:
            assert px is None
    finally:
        dist.destroy_process_group()


def test_render_views_sharded_two_processes():
    import torch

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200.views import orbit_cameras

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    px, ld, st = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert px.shape == (V, H, W, 3) and ld.shape == (V, H, W) and st.shape == (V, 6)
    ds = ab.DeviceScene.from_arrays(_scene_arrays(), 3, "cuda", torch.float32)
    for i, cam in enumerate(orbit_cameras(V, W, H, radius=2.6)):
        res = ab.run_pipeline(ds, cam)
        assert np.array_equal(px[i].view(np.uint32), res.image.pixels.cpu().numpy().view(np.uint32)), i
        assert np.array_equal(ld[i], res.load_map.counts.cpu().numpy()), i
        ls = res.load_stats
        assert int(st[i, 0]) == res.stats.pair_count and int(st[i, 1]) == res.stats.culled_gaussians
        assert int(st[i, 4]) == ls.min and int(st[i, 5]) == ls.max


def test_bench_multi_rank_path_completes():
    """bench.py's multi-rank path (torchrun, two ranks over gloo on cuda:0):
    every loop around a frame transfer or collective runs a rank-agreed
    number of steps, so the run ends (a wall-clock soak loop once left one
    rank's sends unmatched), and rank 0 prints one JSON line with the
    gathered frames counted over both ranks."""
    import json
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ADR_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2",
           "--config", "config1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0

"""CPU: the view-sharded multi-GPU host logic under a real
world_size-2 process group on the gloo backend — view partitioning, the
ragged-slice padding of the frame gather and the view-order reassembly on
rank 0.  On the B200 box the same code runs over NCCL (bench.py --gpus N)."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_views_partition():
    from paper_2409_08669_b200.views import owner_of, shard_views

    for v in (0, 1, 5, 8, 63, 64, 256):
        for world in (1, 2, 3, 4, 8):
            got = [list(shard_views(v, world, r)) for r in range(world)]
            flat = [k for s in got for k in s]
            assert flat == list(range(v)), (v, world)          # disjoint, contiguous, ordered
            sizes = [len(s) for s in got]
            assert max(sizes, default=0) - min(sizes, default=0) <= 1
            for r, s in enumerate(got):
                for k in s:
                    assert owner_of(k, v, world) == r
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def test_pack_unpack_frame_roundtrip():
    from paper_2409_08669_b200.views import pack_frame, unpack_frame

    rng = np.random.default_rng(0)
    px = torch.from_numpy(rng.random((5, 7, 3), dtype=np.float32))
    ld = torch.from_numpy(rng.integers(0, 2**31 - 1, (5, 7), dtype=np.int32))
    f = pack_frame(px, ld)
    p2, l2 = unpack_frame(f)
    assert torch.equal(p2, px) and torch.equal(l2, ld)


def _fake_view(k: int, h: int, w: int):
    """Deterministic per-view frame/stats, a function of the view id only."""
    rng = np.random.default_rng(1000 + k)
    px = torch.from_numpy(rng.random((h, w, 3), dtype=np.float32))
    ld = torch.from_numpy(rng.integers(0, 300, (h, w), dtype=np.int32))
    st = torch.tensor([k * 11, k, int(ld.sum()), int((ld.long() ** 2).sum()), int(ld.min()), int(ld.max())],
                      dtype=torch.int64)
    return px, ld, st


def _worker(rank, world, port, n_views, h, w, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2409_08669_b200.views import gather_frames, pack_frame, shard_views

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = list(shard_views(n_views, world, rank))
        frames, stats = [], []
        for k in mine:
            px, ld, st = _fake_view(k, h, w)
            frames.append(pack_frame(px, ld))
            stats.append(st)
        f = torch.stack(frames) if frames else torch.zeros((0, h, w, 4))
        s = torch.stack(stats) if stats else torch.zeros((0, 6), dtype=torch.int64)
        all_f, all_s = gather_frames(f, s, n_views)
        if rank == 0:
            q.put((all_f.numpy().copy(), all_s.numpy().copy()))
        else:
            assert all_f is None and all_s is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_views,world", [(4, 2), (5, 2), (1, 2), (7, 3)])
def test_gather_frames_gloo(n_views, world):
    """Ragged slices (5 views over 2 ranks, 1 view over 2 ranks, 7 over 3)
    come back on rank 0 only, in view order and bit-identical to the
    per-view single-rank frames."""
    from paper_2409_08669_b200.views import pack_frame

    h, w = 6, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_views, h, w, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_f, got_s = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got_f.shape == (n_views, h, w, 4) and got_s.shape == (n_views, 6)
    for k in range(n_views):
        px, ld, st = _fake_view(k, h, w)
        assert np.array_equal(got_f[k].view(np.uint32), pack_frame(px, ld).numpy().view(np.uint32))
        assert np.array_equal(got_s[k], st.numpy())


def _bcast_worker(rank, world, port, q, dtype_name="float32"):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200.views import broadcast_scene

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        src = None
        dt = getattr(torch, dtype_name)
        if rank == 0:
            a = ab.synthetic_arrays(5, 300, ab.SyntheticSpec(), sh_degree=2, float32=True)
            src = ab.DeviceScene.from_arrays(a, 2, "cpu", dt)
        # only the source knows the dtype; the header makes every rank agree
        ds = broadcast_scene(src, 300, 2, "cpu")
        assert ds.centers.dtype == dt
        q.put((rank, [t.numpy().copy() for t in (ds.centers, ds.scales, ds.rotations, ds.opacities, ds.sh)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype_name", ["float32", "float64"])
def test_broadcast_scene_gloo_world2(dtype_name):
    """Rank 0's scene arrives bit-identical on rank 1 (load once,
    broadcast), whatever dtype the source holds (the header carries it)."""
    import paper_2409_08669_b200 as ab

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q, dtype_name)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    a = ab.synthetic_arrays(5, 300, ab.SyntheticSpec(), sh_degree=2, float32=True)
    want = [np.asarray(x, dtype=dtype_name) for x in (a.centers, a.scales, a.rotations, a.opacities, a.sh)]
    for r in (0, 1):
        for g, w in zip(got[r], want):
            assert g.shape == w.shape and g.dtype == w.dtype and np.array_equal(g, w)

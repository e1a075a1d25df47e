"""Batched frames of one scene (adr_preprocess_views + adr_render_frame_post):
one stage-1 launch for up to 8 views, then each view's stages 2-6.

Every output of every view must equal the single-frame call
(``Rasterizer.launch`` -> adr_render_frame, itself pinned to the reference
and the oracle by test_gpu_parity / test_gpu_fullsize) bit for bit: the
Projection fields, sorted keys and Gaussian indices, tile ranges, image, load
map, load moments and counters.  At full garden size view 0 of the batch is
also checked against the REAL reference's digests (fullsize_digests.json)."""

from __future__ import annotations

import hashlib
import json
import sys

import numpy as np
import pytest

from conftest import GOLDEN, PROJ_FIELDS, ROOT, bits_equal, mixed_spec

pytestmark = pytest.mark.gpu

if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def _snapshot(rast, mode):
    import torch

    torch.cuda.synchronize()
    res = rast.result(mode, rast.proj.alpha_low)
    p = res.pairs.to_numpy()
    out = {f"proj.{k}": v for k, v in res.projection.to_numpy().items() if k in PROJ_FIELDS}
    out.update(keys=p["keys"], gidx=p["gaussian_indices"], ranges=p["tile_ranges"],
               pixels=res.image.pixels.cpu().numpy(), load=res.load_map.counts.cpu().numpy(),
               counters=rast.counters.cpu().numpy(), stats=rast.stats.cpu().numpy())
    return out


def _assert_same(a, b, what):
    assert a.keys() == b.keys()
    for k in a:
        assert bits_equal(a[k], b[k]), f"{what}: {k} differs"


def _cams(n, w, h, radius=3.0):
    from paper_2409_08669_b200.views import orbit_cameras

    return orbit_cameras(n, w, h, radius=radius, background=(0.1, 0.2, 0.3))


def _single(ds, cam, mode, n):
    import paper_2409_08669_b200 as ab

    r = ab.Rasterizer(cam.width, cam.height, n)
    r.render(ds, cam, mode=mode)   # grows the pair buffers until the frame fits
    return _snapshot(r, mode)


def _batched(ds, cams, mode, n, caps):
    """Batched frames; caps[v]: view v's pair capacity (a frame that needs
    more is flagged truncated, never silently cut: asserted here)."""
    import paper_2409_08669_b200 as ab

    rasts = [ab.Rasterizer(c.width, c.height, n, pair_capacity=cap) for c, cap in zip(cams, caps)]
    ab.render_views_batched(ds, cams, rasts, mode=mode)
    out = [_snapshot(r, mode) for r in rasts]
    assert not any(r.truncated() for r in rasts)
    return out


def _check_batch(ds, cams, mode, n):
    singles = [_single(ds, c, mode, n) for c in cams]
    got = _batched(ds, cams, mode, n, [int(s["counters"][0]) + 1024 for s in singles])
    for v in range(len(cams)):
        _assert_same(got[v], singles[v], f"view {v}")
    return got


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("mode", ["baseline", "circle", "aabb"])
def test_batched_views_equal_single_frames(deg, dtype, mode):
    import torch

    import paper_2409_08669_b200 as ab

    n = 30_000
    a = ab.synthetic_arrays(900 + deg, n, mixed_spec(), sh_degree=deg, float32=(dtype == "f32"))
    ds = ab.DeviceScene.from_arrays(a, deg, "cuda", torch.float32 if dtype == "f32" else torch.float64)
    # mixed resolutions in one batch: each view keeps its own tile grid
    cams = _cams(3, 320, 240) + _cams(2, 257, 191, radius=2.2)
    got = _check_batch(ds, cams, mode, n)
    assert any(int(g["counters"][0]) > 0 for g in got)


def test_batched_eight_views_with_wide_grid_view(oracle):
    """A full batch of 8, one view on a > 1024-supertile grid (the path
    without the depth-key extrema plan) and one that sees nothing."""
    import torch

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import Camera

    n = 40_000
    a = ab.synthetic_arrays(77, n, mixed_spec(), sh_degree=3, float32=True)
    ds = ab.DeviceScene.from_arrays(a, 3, "cuda", torch.float32)
    cams = _cams(6, 400, 300)
    cams.append(Camera.from_lookat(position=(0.0, 0.0, -9.0), target=(0.0, 0.0, 0.0), fov_y_deg=60.0,
                                   width=4400, height=4000))   # 68,750 tiles > 1024 supertiles
    cams.append(Camera.from_lookat(position=(0.0, 0.0, 30.0), target=(0.0, 0.0, 60.0), fov_y_deg=60.0,
                                   width=128, height=96))   # looking away: no pairs
    got = _check_batch(ds, cams, "aabb", n)
    assert int(got[-1]["counters"][0]) == 0
    ref = oracle.run_pipeline(dict(centers=a.centers, scales=a.scales, rotations=a.rotations,
                                   opacities=a.opacities, sh=a.sh, sh_degree=3), cams[6], "aabb")
    assert np.array_equal(got[6]["keys"], ref["keys"])
    assert bits_equal(got[6]["pixels"], ref["pixels"])


def test_batched_capacity_overflow_is_reported():
    """A view whose pairs exceed its capacity completes and flags truncation
    (counters[6]) exactly like the single-frame call."""
    import torch

    import paper_2409_08669_b200 as ab

    n = 20_000
    a = ab.synthetic_arrays(5, n, mixed_spec(), sh_degree=1, float32=True)
    ds = ab.DeviceScene.from_arrays(a, 1, "cuda", torch.float32)
    cams = _cams(2, 300, 200)
    rasts = [ab.Rasterizer(c.width, c.height, n, pair_capacity=1000) for c in cams]
    ab.render_views_batched(ds, cams, rasts, mode="aabb")
    torch.cuda.synchronize()
    for r in rasts:
        assert r.truncated() and r.pair_count() > 1000


def test_batched_argument_errors():
    import torch

    import paper_2409_08669_b200 as ab

    n = 1000
    a = ab.synthetic_arrays(6, n, mixed_spec(), sh_degree=0, float32=True)
    ds = ab.DeviceScene.from_arrays(a, 0, "cuda", torch.float32)
    cams = _cams(9, 64, 64)
    rasts = [ab.Rasterizer(64, 64, n) for _ in cams]
    with pytest.raises(ValueError):
        ab.preprocess_views(ds, cams, rasts)            # 9 > MAX_BATCH_VIEWS
    with pytest.raises(ValueError):
        ab.preprocess_views(ds, cams[:2], [rasts[0], rasts[0]])   # shared buffers
    with pytest.raises(ValueError):
        ab.preprocess_views(ds, cams[:2], rasts[:1])
    with pytest.raises(ValueError):
        ab.preprocess_views(ds, cams[:2], [rasts[0], ab.Rasterizer(64, 64, n + 1)])
    with pytest.raises(ValueError):
        ab.preprocess_views(ds, cams[:2], rasts[:2], alpha_low=1.5)


def test_batched_garden_fullsize_matches_reference_digests():
    """configs[2] at full size: 8 views in one stage-1 launch; the batch's
    view of the committed digest hashes to the real reference's outputs, and
    every other view equals its single-frame call."""
    import torch

    import bench
    import paper_2409_08669_b200 as ab

    cfg = bench.CONFIGS["garden"]
    d = json.loads((GOLDEN / "fullsize_digests.json").read_text())["garden"]
    a = bench.scene_arrays(cfg)
    ds = ab.DeviceScene.from_arrays(a, cfg["sh"], "cuda", torch.float32)
    cams = bench.cameras(cfg, 8)
    got = _batched(ds, cams, cfg["mode"], cfg["n"], [int(60e6)] * 8)
    g = got[d["view"]]
    sha = lambda x: hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()  # noqa: E731
    assert int(g["counters"][0]) == d["pairs"] and int(g["counters"][5]) == 0
    for f in PROJ_FIELDS:
        assert sha(g[f"proj.{f}"]) == d["projection"][f], f
    assert sha(g["keys"]) == d["keys"]
    assert sha(g["gidx"].astype(np.int64)) == d["gidx"]
    assert sha(g["ranges"]) == d["ranges"]
    assert sha(g["pixels"]) == d["pixels"]
    assert sha(g["load"]) == d["load"]
    for v in (1, 5, 7):
        _assert_same(got[v], _single(ds, cams[v], cfg["mode"], cfg["n"]), f"garden view {v}")

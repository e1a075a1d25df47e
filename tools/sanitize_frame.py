"""One small fused frame + the stage API + the GPU reference renderer, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_frame.py [N]

With N, one N-Gaussian 640x360 frame instead (multi-block sort / binning).
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2409_08669_b200 as ab  # noqa: E402


def main():
    spec = ab.SyntheticSpec(extent=1.0, scale_range=(0.004, 0.05), anisotropy_range=(1, 5), opacity_range=(0.01, 0.95))
    if len(sys.argv) > 1:   # a multi-block frame: depth-sort look-back chains, many supertile chunks
        n = int(sys.argv[1])
        a = ab.synthetic_arrays(6, n, spec, sh_degree=3, float32=True)
        ds = ab.DeviceScene.from_arrays(a, 3, "cuda", torch.float32)
        cam = ab.Camera.from_lookat((0.3, -0.2, -2.6), (0, 0, 0), width=640, height=360, background=(0.1, 0.2, 0.3))
        res = ab.run_pipeline(ds, cam, mode="aabb")
        ref_img, _ = ab.render_reference(ds, cam)
        torch.cuda.synchronize()
        assert torch.equal(ref_img.pixels.view(torch.int32), res.image.pixels.view(torch.int32))
        cam2 = ab.Camera.from_lookat((-1.2, 0.4, -2.3), (0, 0, 0), width=640, height=360)
        rasts = [ab.Rasterizer(640, 360, n, pair_capacity=2 * res.stats.pair_count + 4096) for _ in range(2)]
        ab.render_views_batched(ds, [cam, cam2], rasts, mode="aabb")   # batched stage 1, multi-block
        torch.cuda.synchronize()
        assert torch.equal(rasts[0].pixels.view(torch.int32), res.image.pixels.view(torch.int32))
        print("sanitize frame OK", n, "Gaussians", res.stats.pair_count, "pairs")
        return
    a = ab.synthetic_arrays(5, 4000, spec, sh_degree=3, float32=True)
    ds = ab.DeviceScene.from_arrays(a, 3, "cuda", torch.float32)
    cam = ab.Camera.from_lookat((0.3, -0.2, -2.6), (0, 0, 0), width=200, height=136, background=(0.1, 0.2, 0.3))
    for mode in ("baseline", "circle", "aabb"):
        res = ab.run_pipeline(ds, cam, mode=mode)
    proj = ab.preprocess(ds, cam)
    grid = ab.TileGrid(200, 136)
    pairs = ab.build_pairs(proj, grid)
    img, lm = ab.render(proj, pairs, grid, cam, ab.ALPHA_LOW, 1e-4)
    ref_img, ref_lm = ab.render_reference(ds, cam)
    rast = ab.Rasterizer(200, 136, len(ds), pair_capacity=500)   # overflow + regrow path
    rast.render(ds, cam)
    torch.cuda.synchronize()
    # batched stage 1 (adr_preprocess_views + adr_render_frame_post): 3 views, one of them
    # with a too-small pair capacity (truncated frame, no out-of-bounds writes)
    cams = [cam, ab.Camera.from_lookat((-1.0, 0.5, -2.2), (0, 0, 0), width=200, height=136),
            ab.Camera.from_lookat((1.5, 0.0, -2.0), (0, 0, 0), width=160, height=120)]
    caps = [res.stats.pair_count + 64, 4 * res.stats.pair_count, 100]
    rasts = [ab.Rasterizer(c.width, c.height, len(ds), pair_capacity=k) for c, k in zip(cams, caps)]
    ab.render_views_batched(ds, cams, rasts, mode="aabb")
    torch.cuda.synchronize()
    assert torch.equal(rasts[0].pixels.view(torch.int32), res.image.pixels.view(torch.int32))
    assert rasts[2].truncated() and not rasts[1].truncated()
    assert torch.equal(ref_img.pixels.view(torch.int32), res.image.pixels.view(torch.int32))
    print("sanitize frame OK", res.stats.pair_count, "pairs")


if __name__ == "__main__":
    main()

"""GPU load-balancing objective: l1_loss / ssim /
total_loss on the GPU vs the real reference's values, and one
toy_balance_step vs the reference's step (tests/golden/toy_golden.npz,
made by tests/golden/make_toy_golden.py).  Tolerances: image terms 1e-12
relative (fp64, summation order differs), losses 1e-10, opacities 1e-12."""

from __future__ import annotations

import time

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def toy():
    with np.load(GOLDEN / "toy_golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("tag", ["a", "b"])
def test_image_terms_match_reference(toy, tag):
    import paper_2409_08669_b200 as ab

    x, y = toy[f"img_{tag}_x"], toy[f"img_{tag}_y"]
    h, w = x.shape[:2]
    ia, ib = ab.Image(w, h, x), ab.Image(w, h, y)
    assert ab.l1_loss(ia, ib) == pytest.approx(float(toy[f"img_{tag}_l1"]), rel=1e-12)
    assert ab.ssim(ia, ib) == pytest.approx(float(toy[f"img_{tag}_ssim"]), rel=1e-12)
    assert ab.psnr(ia, ib) == pytest.approx(float(toy[f"img_{tag}_psnr"]), rel=1e-12)
    assert ab.ssim(ia, ia) == pytest.approx(1.0, abs=1e-12)


def test_total_loss_and_weights():
    import torch

    import paper_2409_08669_b200 as ab

    with pytest.raises(ValueError):
        ab.LossWeights(0.5, 0.5, 0.5)
    with pytest.raises(ValueError):
        ab.LossWeights(-0.1, 0.6, 0.5)
    rng = np.random.default_rng(1)
    a = ab.Image(20, 10, rng.random((10, 20, 3), dtype=np.float32))
    b = ab.Image(20, 10, rng.random((10, 20, 3), dtype=np.float32))
    lm = ab.LoadMap(20, 10, torch.from_numpy(rng.integers(0, 50, (10, 20)).astype(np.int32)).cuda())
    w = ab.DEFAULT_WEIGHTS
    want = w.lambda_l1 * ab.l1_loss(a, b) + w.lambda_ssim * (1.0 - ab.ssim(a, b)) + w.lambda_load * ab.load_loss(lm)
    assert ab.total_loss(a, b, lm) == pytest.approx(want, rel=1e-15)


def test_toy_balance_step_matches_reference(toy):
    import paper_2409_08669_b200 as ab

    n = len(toy["toy_opacities"])
    scene = ab.Scene(gaussians=[ab.Gaussian3D(toy["toy_centers"][i], toy["toy_scales"][i], toy["toy_rotations"][i],
                                              toy["toy_opacities"][i], toy["toy_sh"][i]) for i in range(n)],
                     sh_degree=0)
    cam = ab.Camera(view_matrix=toy["toy_cam_view"], fx=float(toy["toy_cam_fx"]), fy=float(toy["toy_cam_fx"]),
                    width=48, height=40, background=(0.1, 0.1, 0.2))
    reference = ab.Image(48, 40, toy["toy_ref_pixels"])
    res = ab.toy_balance_step(scene, cam, reference, ab.LossWeights(), step=0.05)   # warm-up
    t0 = time.perf_counter()
    res = ab.toy_balance_step(scene, cam, reference, ab.LossWeights(), step=0.05)
    dt = time.perf_counter() - t0
    assert res.loss_before == pytest.approx(float(toy["toy_loss_before"]), rel=1e-10)
    assert res.loss_after == pytest.approx(float(toy["toy_loss_after"]), rel=1e-10)
    got = res.scene.as_arrays().opacities
    assert np.allclose(got, toy["toy_new_opacities"], rtol=0, atol=1e-12)
    print(f"toy step: GPU {dt * 1e3:.1f} ms vs reference {float(toy['toy_ref_seconds']) * 1e3:.0f} ms (CPU)")
    with pytest.raises(ValueError):
        ab.toy_balance_step(scene, cam, reference, ab.LossWeights(), step=0.0)


# -- brute-force reference renderer (sb/oracle.py; §8f row 3) -----------------

@pytest.mark.parametrize("name", ["g_sh3_baseline", "g_sh0_aabb"])
def test_render_reference_matches_golden(name):
    """The reference asserts render_reference == run_pipeline bitwise
    (sb tests/test_oracle.py:58-65); the goldens hold the pipeline's image."""
    from conftest import bits_equal, golden_arrays, golden_camera, load_golden

    import paper_2409_08669_b200 as ab

    g = load_golden(name)
    ds = ab.DeviceScene.from_arrays(golden_arrays(g), int(g["sh_degree"]), "cuda")
    img, lm = ab.render_reference(ds, golden_camera(g))
    assert bits_equal(img.pixels.cpu().numpy(), g["pixels"])
    assert np.array_equal(lm.counts.cpu().numpy(), g["load"])


def test_render_reference_equals_pipeline_fullsize():
    """Large-N self-check with no CPU oracle: the garden-scale frame
    (5.8M Gaussians, 48.8M pairs) through the binning-free path equals the
    fused pipeline bit for bit."""
    import sys

    import torch

    from conftest import ROOT
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    import bench
    import paper_2409_08669_b200 as ab

    cfg = bench.CONFIGS["garden"]
    a = bench.scene_arrays(cfg)
    cam = bench.cameras(cfg, 8)[1]
    ds = ab.DeviceScene.from_arrays(a, cfg["sh"], "cuda", torch.float32)
    res = ab.run_pipeline(ds, cam, mode="aabb")
    img, lm = ab.render_reference(ds, cam)
    assert torch.equal(img.pixels.view(torch.int32), res.image.pixels.view(torch.int32))
    assert torch.equal(lm.counts, res.load_map.counts)

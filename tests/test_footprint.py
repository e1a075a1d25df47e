"""Scalar footprint helpers (paper §4.2-4.3; sb/projection.py:128-289) with
the reference tests' known answers (sb tests/test_projection.py:19-21,
:36-124) and a cross-check of the numpy helpers against the reference
implementation's values on random inputs (generated here by formula)."""

from __future__ import annotations

import math

import numpy as np
import pytest

ALPHA = 1.0 / 255.0


def test_radius_known_answers():
    import paper_2409_08669_b200 as ab

    assert ab.bounding_circle_radius(1.0, 1.0, ALPHA) == pytest.approx(3.3290429691304455, abs=1e-12)
    assert ab.bounding_circle_radius(4.0, 0.1, ALPHA) == pytest.approx(5.090130412603889, abs=1e-12)
    assert ab.bounding_box_halfwidths(np.diag([4.0, 1.0]), 1.0, ALPHA)[0] == pytest.approx(6.658085938260891,
                                                                                           abs=1e-12)
    assert (ab.radius_baseline(1.0), ab.radius_baseline(4.0), ab.radius_baseline(2.0)) == (3, 6, 5)
    assert ab.radius_adaptive(1.0, ALPHA, ALPHA) is None
    assert ab.radius_adaptive(1.0, 1.0, ALPHA) == 3
    assert ab.radius_adaptive(4.0, 0.4, ALPHA) == 6      # ceil applied after the min
    assert ab.radius_adaptive(4.0, 0.1, ALPHA) == 6
    assert ab.aabb_extents(np.diag([4.0, 1.0]), 1.0, ALPHA, 4.0) == (6, 4)
    assert ab.aabb_extents(np.diag([4.0, 1.0]), ALPHA, ALPHA, 4.0) is None


def test_covariance_and_eigen():
    import paper_2409_08669_b200 as ab

    assert np.allclose(ab.build_covariance3d((1, 1, 1), (1, 0, 0, 0)), np.eye(3), atol=1e-12)
    h = math.sqrt(0.5)
    assert np.allclose(ab.build_covariance3d((1, 2, 3), (h, 0, 0, h)), np.diag([4.0, 1.0, 9.0]), atol=1e-12)
    with pytest.raises(ValueError):
        ab.build_covariance3d((1, float("nan"), 1), (1, 0, 0, 0))
    with pytest.raises(ValueError):
        ab.build_covariance3d((1, 0, 1), (1, 0, 0, 0))
    assert ab.eigen_extents(np.diag([2.0, 1.0])) == (2.0, 1.0)
    lmax, lmin = ab.eigen_extents(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert (lmax, lmin) == (pytest.approx(3.0, abs=1e-12), pytest.approx(1.0, abs=1e-12))
    with pytest.raises(ValueError):
        ab.eigen_extents(np.array([[1.0, 2.0], [2.0, 1.0]]))
    rng = np.random.default_rng(0)
    for _ in range(50):
        l1 = rng.uniform(0.5, 60)
        l2 = l1 / rng.uniform(1, 20)
        t = rng.uniform(0, 2 * math.pi)
        r = np.array([[math.cos(t), -math.sin(t)], [math.sin(t), math.cos(t)]])
        cov = r @ np.diag([l1, l2]) @ r.T
        assert np.allclose(sorted(ab.eigen_extents(cov)), np.linalg.eigvalsh(cov), rtol=1e-10)


def test_ellipse_coefficients_and_containment():
    import paper_2409_08669_b200 as ab

    e = ab.ellipse_coefficients(np.eye(2), math.e * ALPHA, ALPHA)
    assert (e.a, e.b, e.c) == (1.0, 1.0, -0.0) and e.d == pytest.approx(-2.0, abs=1e-12)
    rng = np.random.default_rng(4)
    for _ in range(200):  # every boundary point lies inside the AABB half-widths
        cov = np.array([[rng.uniform(1, 30), 0.0], [0.0, rng.uniform(1, 30)]])
        cov[0, 1] = cov[1, 0] = rng.uniform(-0.9, 0.9) * math.sqrt(cov[0, 0] * cov[1, 1])
        sigma = rng.uniform(0.05, 1.0)
        hx, hy = ab.bounding_box_halfwidths(cov, sigma, ALPHA)
        c = ab.ellipse_coefficients(cov, sigma, ALPHA)
        lmax, _ = ab.eigen_extents(cov)
        r = ab.bounding_circle_radius(lmax, sigma, ALPHA)
        th = rng.uniform(0, 2 * math.pi)
        # boundary point along direction th: solve a x^2 + b y^2 + c x y + d = 0
        dx, dy = math.cos(th), math.sin(th)
        q = c.a * dx * dx + c.b * dy * dy + c.c * dx * dy
        t = math.sqrt(-c.d / q)
        assert abs(t * dx) <= hx * (1 + 1e-9) and abs(t * dy) <= hy * (1 + 1e-9) and t <= r * (1 + 1e-9)


def test_evaluate_sh_degree0_and_clip():
    import paper_2409_08669_b200 as ab

    rgb = np.array([0.2, 0.5, 0.9])
    dc = (rgb - 0.5) / ab.footprint.SH_C0
    assert np.allclose(ab.evaluate_sh(dc[None, :], (0, 0, 1), 0), rgb, atol=1e-12)
    assert np.array_equal(ab.evaluate_sh(np.full((1, 3), 10.0), (0, 0, 1), 0), np.ones(3))
    with pytest.raises(ValueError):
        ab.evaluate_sh(np.zeros((4, 3)), (0, 0, 1), 2)


@pytest.mark.gpu
def test_project_gaussian_and_composite_pixels_vs_pipeline():
    """project_gaussian = row of the batched GPU preprocess; the host
    composite_pixels over a tile's span = the GPU render of that tile."""
    import torch

    import paper_2409_08669_b200 as ab
    from conftest import make_camera, mixed_spec

    cam = make_camera(width=48, height=32, background=(0.1, 0.2, 0.3))
    scene = ab.generate_synthetic(5, 40, mixed_spec())
    res = ab.run_pipeline(scene, cam, mode="aabb")
    proj = res.projection.to_numpy()
    for i, g in enumerate(scene.gaussians[:10]):
        pg = ab.project_gaussian(g, cam)
        if pg is None:
            assert not proj["valid"][i]
            continue
        assert np.array_equal(pg.mean2d, proj["mean2d"][i].astype(np.float64))
        assert (pg.extent.rx, pg.extent.ry) == (proj["ext_x"][i], proj["ext_y"][i])
    p = res.pairs.to_numpy()
    t = 4  # one tile
    lo, hi = p["tile_ranges"][t]
    tx, ty = t % 3, t // 3
    xs, ys = np.meshgrid(np.arange(16 * tx, 16 * tx + 16), np.arange(16 * ty, 16 * ty + 16))
    rgb, cnt = ab.composite_pixels(xs.ravel(), ys.ravel(), p["gaussian_indices"][lo:hi], proj, ab.ALPHA_LOW,
                                   cam.background)
    img = res.image.pixels.cpu().numpy()[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16].reshape(-1, 3)
    assert np.array_equal(rgb.view(np.uint32), img.view(np.uint32))
    assert np.array_equal(cnt, res.load_map.counts.cpu().numpy()[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16].ravel())

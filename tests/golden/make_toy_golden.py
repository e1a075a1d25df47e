"""Golden fixtures for SURVEY.md §8f row 1 (the load-balancing loss path):
the REAL reference's l1_loss / ssim / total_loss on fixed images and one
toy_balance_step on a seeded scene (sb/metrics.py:94-210).

    python tests/golden/make_toy_golden.py      (build container only)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists():
        sys.path.insert(0, str(p))
        break

import splatbench as sb  # noqa: E402
from splatbench import metrics as sbm  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    out = {}
    # image losses on fixed random images (odd sizes exercise the zero-padded borders)
    rng = np.random.default_rng(12)
    for tag, (h, w) in {"a": (37, 53), "b": (64, 64)}.items():
        x = rng.random((h, w, 3), dtype=np.float32)
        y = np.clip(x + rng.normal(0, 0.1, (h, w, 3)).astype(np.float32), 0, 1).astype(np.float32)
        ia, ib = sb.Image(w, h, x), sb.Image(w, h, y)
        out[f"img_{tag}_x"], out[f"img_{tag}_y"] = x, y
        out[f"img_{tag}_l1"] = sbm.l1_loss(ia, ib)
        out[f"img_{tag}_ssim"] = sbm.ssim(ia, ib)
        out[f"img_{tag}_psnr"] = sbm.psnr(ia, ib)
    # one toy_balance_step (SH0, <= 500 Gaussians)
    spec = sb.SyntheticSpec(extent=0.8, scale_range=(0.02, 0.07), anisotropy_range=(1.0, 3.0),
                            opacity_range=(0.05, 0.95))
    scene = sb.generate_synthetic(31, 48, spec)
    cam = sb.Camera.from_lookat((0.1, 0.2, -3.0), (0, 0, 0), width=48, height=40, background=(0.1, 0.1, 0.2))
    target_scene = sb.generate_synthetic(32, 48, spec)
    reference = sb.run_pipeline(target_scene, cam).image
    weights = sbm.LossWeights()
    t = time.perf_counter()
    res = sbm.toy_balance_step(scene, cam, reference, weights, step=0.05)
    dt = time.perf_counter() - t
    a = scene.as_arrays()
    out.update(toy_centers=a.centers, toy_scales=a.scales, toy_rotations=a.rotations, toy_opacities=a.opacities,
               toy_sh=a.sh, toy_cam_view=cam.view_matrix, toy_cam_fx=cam.fx, toy_ref_pixels=reference.pixels,
               toy_loss_before=res.loss_before, toy_loss_after=res.loss_after,
               toy_new_opacities=res.scene.as_arrays().opacities, toy_ref_seconds=dt)
    np.savez_compressed(OUT / "toy_golden.npz", **out)
    print("wrote", OUT / "toy_golden.npz", f"(reference toy step {dt:.2f} s)", res.loss_before, res.loss_after)


if __name__ == "__main__":
    main()

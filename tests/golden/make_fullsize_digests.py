"""sha256 digests of the REAL reference (splatbench 0.1.0) at BASELINE.json's
full sizes — configs[1] truck, configs[2] garden, configs[3] playroom and
configs[4] stress, one orbit view each — for tests/test_gpu_fullsize.py.

Run in the build container (the reference is importable here, not on the GPU
box); a 5.8M frame takes ~2 min on 8 cores plus ~40 s of scene construction:

    python tests/golden/make_fullsize_digests.py [name ...]

Inputs are regenerated on both sides by bench.scene_arrays / bench.cameras
(seeded draws identical to sb.generate_synthetic + SH rest N(0, 0.3^2),
rounded to fp32); the inputs' own digest is stored so a drift in the
generator is caught before any output is compared.  Output digests cover the
sorted keys, Gaussian indices (int64), tile ranges, image, load map and all
ten Projection fields, plus P, the culled count and load_loss.
"""

from __future__ import annotations

import gc
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists():
        sys.path.insert(0, str(p))
        break
sys.path.insert(0, str(ROOT))

import splatbench as sb  # noqa: E402

import bench  # noqa: E402

OUT = Path(__file__).resolve().parent / "fullsize_digests.json"
CASES = {"truck": 3, "garden": 0, "playroom": 5, "stress": 0}
PROJ_FIELDS = ("valid", "mean2d", "cov2d", "conic", "depth", "color", "opacity", "lambda_max",
               "ext_x", "ext_y")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def inputs_sha(a) -> str:
    h = hashlib.sha256()
    for arr in (a.centers, a.scales, a.rotations, a.opacities, a.sh):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def case(name: str, view: int) -> dict:
    cfg = bench.CONFIGS[name]
    a = bench.scene_arrays(cfg)
    cam = bench.cameras(cfg, 8)[view]
    t0 = time.time()
    gs = [sb.Gaussian3D(center=a.centers[i], scale=a.scales[i], rotation=a.rotations[i],
                        opacity=a.opacities[i], sh_coeffs=a.sh[i]) for i in range(cfg["n"])]
    scene = sb.Scene(gaussians=gs, sh_degree=cfg["sh"])
    t1 = time.time()
    res = sb.run_pipeline(scene, cam, mode=sb.CullingMode(cfg["mode"]), threads=os.cpu_count() or 1)
    t2 = time.time()
    p = res.projection
    rec = {
        "view": view, "mode": cfg["mode"], "inputs_sha256": inputs_sha(a),
        "view_matrix": np.asarray(cam.view_matrix).tolist(),
        "pairs": len(res.pairs), "culled": res.stats.culled_gaussians,
        "keys": sha(res.pairs.keys), "gidx": sha(res.pairs.gaussian_indices.astype(np.int64)),
        "ranges": sha(res.pairs.tile_ranges), "pixels": sha(res.image.pixels),
        "load": sha(res.load_map.counts), "load_loss": sb.load_loss(res.load_map),
        "projection": {f: sha(getattr(p, f)) for f in PROJ_FIELDS},
        "reference_seconds": {"scene_build": round(t1 - t0, 1), "run_pipeline": round(t2 - t1, 1),
                              "threads": os.cpu_count()},
    }
    print(f"{name} view {view}: P={rec['pairs']} culled={rec['culled']} "
          f"build {t1 - t0:.0f}s frame {t2 - t1:.0f}s", flush=True)
    del gs, scene, res, p
    gc.collect()
    return rec


def main(names):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in names:
        data[name] = case(name, CASES[name])
        OUT.write_text(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))

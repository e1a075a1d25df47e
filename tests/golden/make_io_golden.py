"""Golden fixtures for the host-side I/O rows,
generated from the REAL reference (splatbench 0.1.0) in the build container:

    python tests/golden/make_io_golden.py

* io_scene_sh3.ply     — sb.save_ply of a seeded SH3 scene (raw PLY bytes)
* io_golden.npz        — sb.load_ply of that file (activated arrays), the
                         reference's JSON/PPM/PNG/PGM bytes' sha256, and the
                         gen-scene output digests
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if p.exists():
        sys.path.insert(0, str(p))
        break

import splatbench as sb  # noqa: E402
from splatbench import imageio as sbio  # noqa: E402
from splatbench import scene as sbs  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(path) -> str:
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


def main():
    rng = np.random.default_rng(77)
    n, deg = 40, 3
    k = (deg + 1) ** 2
    gs = []
    for i in range(n):
        q = rng.normal(size=4)
        gs.append(sb.Gaussian3D(center=rng.uniform(-1, 1, 3), scale=rng.uniform(0.01, 0.1, 3),
                                rotation=q / np.linalg.norm(q), opacity=float(rng.uniform(0.02, 0.98)),
                                sh_coeffs=rng.normal(0, 0.4, (k, 3))))
    scene = sb.Scene(gaussians=gs, sh_degree=deg)
    ply = OUT / "io_scene_sh3.ply"
    sbs.save_ply(scene, ply)
    back = sbs.load_ply(ply)
    a = back.as_arrays()
    o = scene.as_arrays()
    out = dict(ply_centers=a.centers, ply_scales=a.scales, ply_rotations=a.rotations,
               ply_opacities=a.opacities, ply_sh=a.sh, ply_sh_degree=back.sh_degree,
               ply_sha=sha(ply), orig_centers=o.centers, orig_scales=o.scales, orig_rotations=o.rotations,
               orig_opacities=o.opacities, orig_sh=o.sh)
    with tempfile.TemporaryDirectory() as td:
        sbs.save_ply(back, Path(td) / "r.ply")
        out["resave_sha"] = sha(Path(td) / "r.ply")
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        sbs.save_json(scene, td / "s.json")
        out["json_sha"] = sha(td / "s.json")
        js = sbs.load_json(td / "s.json").as_arrays()
        out["json_centers"] = js.centers
        out["json_rotations"] = js.rotations
        # image writers on a fixed image / load map
        pix = np.clip(np.random.default_rng(5).random((13, 17, 3), dtype=np.float32) * 1.2 - 0.1, -0.1, 1.1)
        pix = pix.astype(np.float32)
        img = sb.Image(width=17, height=13, pixels=pix)
        counts = np.random.default_rng(6).integers(0, 70000, (13, 17)).astype(np.int32)
        lm = sb.LoadMap(width=17, height=13, counts=counts)
        sbio.write_png(img, td / "i.png")
        sbio.write_ppm(img, td / "i.ppm")
        sbio.write_pgm16(lm, td / "l.pgm")
        sbio.write_loadmap_png(lm, td / "l.png")
        out.update(img_pixels=pix, load_counts=counts, png_sha=sha(td / "i.png"), ppm_sha=sha(td / "i.ppm"),
                   pgm_sha=sha(td / "l.pgm"), loadpng_sha=sha(td / "l.png"))
        # gen-scene through the reference CLI's own generator + writers
        syn = sb.generate_synthetic(9, 25, sb.SyntheticSpec())
        sbs.save_scene(syn, td / "g.json")
        sbs.save_scene(syn, td / "g.ply")
        out["gen_json_sha"] = sha(td / "g.json")
        out["gen_ply_sha"] = sha(td / "g.ply")
        # camera sidecar parsing (cli.load_camera) -> view matrix / focal
        cam_doc = {"position": [0.3, -0.2, -3.0], "target": [0, 0, 0], "fov_y_deg": 50, "width": 64,
                   "height": 48, "background": [0.1, 0.2, 0.3]}
        # (splatbench.cli imports matplotlib, absent here: restate cli.py:45-68)
        cam = sb.Camera.from_lookat(position=cam_doc["position"], target=cam_doc["target"],
                                    up=cam_doc.get("up", (0.0, 1.0, 0.0)), fov_y_deg=float(cam_doc["fov_y_deg"]),
                                    width=int(cam_doc["width"]), height=int(cam_doc["height"]),
                                    near_plane=float(cam_doc.get("near", 0.2)),
                                    background=cam_doc.get("background", (0.0, 0.0, 0.0)))
        out.update(cam_doc=json.dumps(cam_doc), cam_view_matrix=cam.view_matrix, cam_fx=cam.fx)
    np.savez_compressed(OUT / "io_golden.npz", **out)
    print("wrote", OUT / "io_golden.npz", ply)


if __name__ == "__main__":
    main()

"""Fraction of Gaussians that touch >= 1 tile (counters[2]) per bench view."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import bench
import paper_2409_08669_b200 as ab

for name in sys.argv[1:] or ["garden", "truck", "playroom", "stress"]:
    cfg = bench.CONFIGS[name]
    ds = ab.DeviceScene.from_arrays(bench.scene_arrays(cfg), cfg["sh"], "cuda", torch.float32)
    rast = ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"])
    fr = []
    for cam in bench.cameras(cfg, 8):
        res = rast.render(ds, cam, mode=cfg["mode"])
        fr.append(int(rast.counters[2].item()) / cfg["n"])
    print(name, "selected fraction per view", [round(f, 3) for f in fr], flush=True)
    del ds, rast
    torch.cuda.empty_cache()

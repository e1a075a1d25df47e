"""Per-view stage times (single-frame path, CUDA events) and pair counts of the bench views."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import bench
import paper_2409_08669_b200 as ab

name = sys.argv[1] if len(sys.argv) > 1 else "garden"
cfg = bench.CONFIGS[name]
ds = ab.DeviceScene.from_arrays(bench.scene_arrays(cfg), cfg["sh"], "cuda", torch.float32)
rast = ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"])
for v, cam in enumerate(bench.cameras(cfg, 8)):
    rast.render(ds, cam, mode=cfg["mode"])
    res = rast.render(ds, cam, mode=cfg["mode"])
    st = {k: round(x * 1e3, 3) for k, x in res.stats.stage_seconds().items()}
    print(name, "view", v, "pairs", res.stats.pair_count, "load mean/max", round(res.load_stats.mean, 1),
          res.load_stats.max, st, flush=True)

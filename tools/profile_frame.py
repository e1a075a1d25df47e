"""Render one bench frame between cudaProfilerStart/Stop so ncu can capture
exactly that frame's kernels:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/profile_frame.py --config garden
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2409_08669_b200 as ab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="garden")
    ap.add_argument("--frames", type=int, default=1)
    ap.add_argument("--batch", type=int, default=0,
                    help="profile one bench step instead: N views through one preprocess_views launch "
                         "+ each view's stages 2-6 (one stream, serialised)")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    arrays = bench.scene_arrays(cfg)
    ds = ab.DeviceScene.from_arrays(arrays, cfg["sh"], "cuda", torch.float32)
    cam = bench.cameras(cfg, bench.VIEWS_PER_RANK)[0]
    rast = ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"])
    res = rast.render(ds, cam, mode=cfg["mode"])
    rast.fit_capacity(res.stats.pair_count)
    res = rast.render(ds, cam, mode=cfg["mode"])
    print("pairs", res.stats.pair_count, "stages_ms",
          {k: round(v * 1e3, 4) for k, v in res.stats.stage_seconds().items()}, flush=True)
    torch.cuda.synchronize()
    if a.batch > 0:
        cams = bench.cameras(cfg, bench.VIEWS_PER_RANK)[:a.batch]
        rasts = [rast] + [ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"], pair_capacity=rast.cap, timing=False)
                          for _ in cams[1:]]
        for r in rasts:   # size every view's pair buffers
            r.fit_capacity(int(res.stats.pair_count * 1.1))
        ab.render_views_batched(ds, cams, rasts, mode=cfg["mode"])
        torch.cuda.synchronize()
        assert not any(r.truncated() for r in rasts)
        torch.cuda.profiler.start()
        ab.render_views_batched(ds, cams, rasts, mode=cfg["mode"])
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    torch.cuda.profiler.start()
    for _ in range(a.frames):
        rast.launch(ds, cam, mode=cfg["mode"])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()

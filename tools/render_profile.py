"""Warp-iteration outcome counters of k_render for one frame (the counting
instantiation selected at run time by adr_render_selfcheck):

    python tools/render_profile.py --config garden
"""

from __future__ import annotations

import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2409_08669_b200 as ab  # noqa: E402
from paper_2409_08669_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="garden")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    ds = ab.DeviceScene.from_arrays(bench.scene_arrays(cfg), cfg["sh"], "cuda", torch.float32)
    cam = bench.cameras(cfg, bench.VIEWS_PER_RANK)[0]
    rast = ab.Rasterizer(cfg["w"], cfg["h"], cfg["n"])
    res = rast.render(ds, cam, mode=cfg["mode"])
    rast.fit_capacity(res.stats.pair_count)
    L = _lib.lib()
    out = (ctypes.c_ulonglong * 8)()
    L.adr_render_selfcheck(1, None)          # reset, counting instantiation on
    res = rast.render(ds, cam, mode=cfg["mode"])
    torch.cuda.synchronize()
    L.adr_render_selfcheck(0, out)
    it, tau_fail, alpha_fail, live, ptau, pcontrib, batches, tau_fail_nodone = (int(out[i]) for i in range(8))
    P = res.stats.pair_count
    unsafe, batches = divmod(batches, 1000000000)
    print(f"pairs {P}  batches(warp) {batches}")
    print(f"warp iterations {it}  ({it / P:.3f} per pair; 4 would be every quadrant)")
    print(f"  all lanes fail tau   {tau_fail} ({tau_fail / it:.1%})")
    print(f"    ... with no done pixel in the warp {tau_fail_nodone} ({tau_fail_nodone / it:.1%})")
    print(f"  removed by quad_mask {alpha_fail} ({alpha_fail / it:.1%})  unsafe removals {unsafe}")
    print(f"  live pixels / iteration    {live / it:.1f} of 64")
    print(f"  pixels passing tau / it    {ptau / it:.1f}")
    print(f"  pixels contributing / it   {pcontrib / it:.1f}   (load-map total {int(res.load_map.counts.long().sum())})")


if __name__ == "__main__":
    main()

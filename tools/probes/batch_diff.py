"""Debug: where batched frames differ from single frames."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
import numpy as np
import torch
import paper_2409_08669_b200 as ab
from conftest import mixed_spec
from paper_2409_08669_b200.views import orbit_cameras

for mode in ["baseline", "circle", "aabb"]:
    n = 30000
    a = ab.synthetic_arrays(900, n, mixed_spec(), sh_degree=0, float32=True)
    ds = ab.DeviceScene.from_arrays(a, 0, "cuda", torch.float32)
    cams = orbit_cameras(3, 320, 240, radius=3.0)
    rb = [ab.Rasterizer(320, 240, n) for _ in cams]
    ab.render_views_batched(ds, cams, rb, mode=mode)
    torch.cuda.synchronize()
    for v, c in enumerate(cams):
        rs = ab.Rasterizer(320, 240, n)
        rs.render(ds, c, mode=mode)
        torch.cuda.synchronize()
        pb = rb[v].result(mode, 0.0039215686).pairs.to_numpy()
        ps = rs.result(mode, 0.0039215686).pairs.to_numpy()
        kb, ks = pb["keys"], ps["keys"]
        print(mode, v, "P", len(kb), len(ks), "ctr", rb[v].counters.cpu().tolist(), rs.counters.cpu().tolist())
        if len(kb) == len(ks):
            d = np.nonzero(kb != ks)[0]
            print("  key diffs", len(d), d[:5], [hex(int(x)) for x in kb[d[:3]]], [hex(int(x)) for x in ks[d[:3]]])
            print("  gidx equal", np.array_equal(pb["gaussian_indices"], ps["gaussian_indices"]),
                  "ranges equal", np.array_equal(pb["tile_ranges"], ps["tile_ranges"]),
                  "pix equal", torch.equal(rb[v].pixels, rs.pixels))

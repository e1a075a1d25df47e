import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2409_08669_b200 as ab
mixed_spec = lambda: ab.SyntheticSpec(extent=1.2, scale_range=(0.01, 0.06), anisotropy_range=(1.0, 6.0), opacity_range=(0.01, 1.0))
a = ab.synthetic_arrays(17, 4000, mixed_spec(), sh_degree=0, float32=True)
cam = ab.Camera.from_lookat((0, 0, -3), (0, 0, 0), width=2200, height=2000)
res = ab.run_pipeline(ab.DeviceScene.from_arrays(a, 0, "cuda", torch.float32), cam)
torch.cuda.synchronize(); print("ok", res.stats.pair_count)

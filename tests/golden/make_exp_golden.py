"""Golden vectors for numpy's float32 exp (the reference's np.exp at
sb/render.py:96), generated with numpy in the build container:

    python tests/golden/make_exp_golden.py

Stores float32 input bits and np.exp output bits for a stratified sample of
the range the render loop reaches ([-104.5, 1]) plus edge cases, so the exp
restatement (oracle + GPU) is pinned on hosts whose numpy dispatches a
different exp implementation.
"""
from pathlib import Path

import numpy as np

rng = np.random.default_rng(2409)
lo, hi = np.float32(-104.5).view(np.uint32), np.float32(1.0).view(np.uint32)
neg = rng.integers(0x80000000, int(lo) + 1, 60000, dtype=np.uint64).astype(np.uint32)  # [-104.5, -0]
pos = rng.integers(0, int(hi) + 1, 10000, dtype=np.uint64).astype(np.uint32)          # [0, 1]
edge = np.array([0x00000000, 0x80000000, 0x7f800000, 0xff800000, 0x7fc00000,
                 np.float32(88.72283935546875).view(np.uint32),
                 np.float32(88.7228470).view(np.uint32),
                 np.float32(-103.97208404541015625).view(np.uint32),
                 np.float32(-103.9720916748046875).view(np.uint32),
                 np.float32(-87.33654).view(np.uint32), np.float32(-0.5).view(np.uint32)],
                dtype=np.uint32)
x = np.concatenate([neg, pos, edge]).view(np.float32)
with np.errstate(over="ignore"):
    y = np.exp(x)
np.savez_compressed(Path(__file__).resolve().parent / "exp_np_f32.npz",
                    x_bits=x.view(np.uint32), y_bits=y.view(np.uint32))
print(len(x), "vectors")

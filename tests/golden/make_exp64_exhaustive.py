"""Exhaustive pin of the PLY loader's float64 activations (sb/scene.py:385-386:
scipy.special.expit for opacity, np.exp for scales), generated with numpy /
scipy in the build container:

    python tests/golden/make_exp64_exhaustive.py

A PLY stores float32, so the inputs are every non-NaN float32 bit pattern u
widened to float64.  For each function f and range [lo, hi) of patterns it
stores H = sum of (bits64(f(u)) + 1) * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64
(order-independent; any changed output bit changes it).  The oracle
(tests/test_oracle_golden.py, the named sub-ranges) and the GPU
(tests/test_gpu_ply.py, all 2^32) reproduce numpy / scipy exactly when they
reproduce H.  NaN inputs are skipped: the loader rejects non-finite rows
before activating (sb/scene.py:370-373).
"""
import json
import platform
from pathlib import Path

import numpy as np
import scipy
from scipy.special import expit

K = np.uint64(0x9E3779B97F4A7C15)
CHUNK = 1 << 25


def f32_bits(v: float) -> int:
    return int(np.float32(v).view(np.uint32))


RANGES = {
    "all_2p32": (0, 1 << 32),
    "pos_half": (f32_bits(0.5), f32_bits(0.75)),
    "neg_small": (f32_bits(-0.0), f32_bits(-8.0)),
    "pos_rare": (f32_bits(700.0), f32_bits(1100.0)),
    "neg_rare": (f32_bits(-500.0), f32_bits(-1100.0)),
}


def checksum(fn, lo: int, hi: int) -> int:
    total = np.uint64(0)
    with np.errstate(all="ignore"):
        for a in range(lo, hi, CHUNK):
            u = np.arange(a, min(a + CHUNK, hi), dtype=np.uint64)
            x = u.astype(np.uint32).view(np.float32)
            keep = ~np.isnan(x)
            y = fn(x[keep].astype(np.float64)).view(np.uint64)
            total += np.sum((y + np.uint64(1)) * ((u[keep] * K) | np.uint64(1)), dtype=np.uint64)
    return int(total)


def main():
    out = {}
    for name, fn in (("exp", np.exp), ("expit", expit)):
        out[name] = {k: checksum(fn, lo, hi) for k, (lo, hi) in RANGES.items()}
        print(name, out[name], flush=True)
    out["ranges"] = {k: [lo, hi] for k, (lo, hi) in RANGES.items()}
    out["numpy"], out["scipy"], out["machine"] = np.__version__, scipy.__version__, platform.machine()
    out["libc"] = platform.libc_ver()
    (Path(__file__).resolve().parent / "exp64_exhaustive.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

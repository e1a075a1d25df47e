"""Exhaustive pin of numpy's float32 exp (the reference's np.exp at
sb/render.py:96), generated with numpy in the build container:

    python tests/golden/make_exp_exhaustive.py

Over every float32 bit pattern u (all 2^32, including signed zeros,
subnormals, infinities and NaNs) and over the render's fast-path range
[-87, 88], stores H = sum of (y + 1) * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64,
y = the bits of np.exp(float32(u)).  The sum is order-independent and every
changed output bit changes it, so the C oracle (tests/test_oracle_golden.py)
and the GPU's exp_np (tests/test_gpu_parity.py) reproduce numpy's exp on ALL
inputs exactly when they reproduce H.  Also records numpy's version and
SIMD dispatch for provenance.
"""
import json
import platform
from pathlib import Path

import numpy as np

K = np.uint64(0x9E3779B97F4A7C15)
CHUNK = 1 << 26


def checksum(lo: int, hi: int) -> int:
    total = np.uint64(0)
    with np.errstate(over="ignore", invalid="ignore"):
        for a in range(lo, hi, CHUNK):
            u = np.arange(a, min(a + CHUNK, hi), dtype=np.uint64)
            y = np.exp(u.astype(np.uint32).view(np.float32)).view(np.uint32).astype(np.uint64)
            total += np.sum((y + np.uint64(1)) * ((u * K) | np.uint64(1)), dtype=np.uint64)
    return int(total)


def main():
    lo87 = int(np.float32(-87.0).view(np.uint32))      # [-87, -0]: patterns 0x80000000 .. bits(-87)
    hi88 = int(np.float32(88.0).view(np.uint32))       # [+0, 88]: patterns 0 .. bits(88)
    out = {
        "all_2p32": checksum(0, 1 << 32),
        "range_m87_88": (checksum(0, hi88 + 1) + checksum(0x80000000, lo87 + 1)) % (1 << 64),
        "numpy": np.__version__,
        "machine": platform.machine(),
        "simd": [k for k, v in np._core._multiarray_umath.__cpu_features__.items() if v and "AVX512" in k]
        if hasattr(np, "core") else [],
    }
    (Path(__file__).resolve().parent / "exp_exhaustive.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()

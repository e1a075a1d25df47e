"""Deterministic PLY checkpoints for the device-ingest parity tests
(tests/test_gpu_ply.py) and their reference digests
(tests/golden/make_ply_golden.py).  numpy's Generator streams are
platform-independent, so the files are byte-identical on every machine."""
from __future__ import annotations

from pathlib import Path

import numpy as np

CASES = {
    # name: (sh_degree, rows, property order, extra properties)
    "sh3_extreme": (3, 200_003, "standard", ("extra_a", "extra_b")),
    "sh0_shuffled": (0, 1_001, "shuffled", ("w_extra",)),
    "sh1_small": (1, 517, "standard", ()),
    "sh2_reversed": (2, 4_099, "reversed", ()),
}


def _names(deg: int) -> list:
    rest = 3 * ((deg + 1) ** 2 - 1)
    return (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
            + [f"f_rest_{i}" for i in range(rest)]
            + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])


def _extreme(rng, n: int, lo: float, hi: float) -> np.ndarray:
    """Mixture: typical values, uniform over [lo, hi], and fixed edge values
    (the exp / expit special-case thresholds)."""
    v = rng.normal(0.0, 3.0, n)
    pick = rng.random(n)
    v = np.where(pick < 0.3, rng.uniform(lo, hi, n), v)
    edges = np.array([0.0, -0.0, 512.0, -512.0, 707.7, -707.7, 708.4, -708.4, 709.78, -709.78,
                      744.5, -744.5, 745.2, -745.2, 1000.0, -1000.0, 3e38, -3e38, 1e-30, -1e-30,
                      2.0 ** -60, 88.7, -103.9], dtype=np.float64)
    idx = rng.choice(n, size=min(n, 4 * edges.size), replace=False)
    v[idx] = np.resize(edges, idx.size)
    return v.astype(np.float32)


def make_raw(name: str):
    """-> (property names in file order, (rows, P) float32 matrix)."""
    deg, n, order, extra = CASES[name]
    rng = np.random.default_rng(abs(hash_name(name)))
    names = _names(deg)
    cols = {nm: rng.normal(0.0, 1.0, n).astype(np.float32) for nm in names}
    for c in ("x", "y", "z"):
        cols[c] = (rng.normal(0.0, 10.0, n)).astype(np.float32)
    cols["opacity"] = _extreme(rng, n, -1100.0, 1100.0)
    for c in ("scale_0", "scale_1", "scale_2"):
        cols[c] = _extreme(rng, n, -760.0, 720.0)
    q = rng.normal(0.0, 1.0, (n, 4)) * np.exp(rng.normal(0.0, 4.0, (n, 1)))
    for i in range(4):
        cols[f"rot_{i}"] = q[:, i].astype(np.float32)
    for nm in extra:
        cols[nm] = rng.normal(0.0, 1.0, n).astype(np.float32)
    order_names = names + list(extra)
    if order == "shuffled":
        order_names = [order_names[i] for i in rng.permutation(len(order_names))]
    elif order == "reversed":
        order_names = order_names[::-1]
    return order_names, np.stack([cols[nm] for nm in order_names], axis=1)


def hash_name(name: str) -> int:
    h = 1469598103934665603
    for ch in name.encode():
        h = ((h ^ ch) * 1099511628211) % (1 << 63)
    return h


def write_ply(path: Path, names, raw: np.ndarray) -> Path:
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {raw.shape[0]}"]
    head += [f"property float {nm}" for nm in names] + ["end_header"]
    path = Path(path)
    path.write_bytes(("\n".join(head) + "\n").encode("ascii") + np.ascontiguousarray(raw, dtype="<f4").tobytes())
    return path


def write_case(dirpath: Path, name: str) -> Path:
    names, raw = make_raw(name)
    return write_ply(Path(dirpath) / f"{name}.ply", names, raw)

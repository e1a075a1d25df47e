"""Device-side PLY ingest on one B200 (sb/scene.py:316-398 load_ply, §8(f) row 4).

Writes a synthetic SH-3 checkpoint of N Gaussians (default: garden's 5.8M,
62 float32 properties per row, 1.44 GB) to a temp dir, then times
  * kernel : adr_ply_activate on a device-resident raw matrix (CUDA events,
             warm, L2 flushed between launches by the size itself) -> GB/s of
             algorithmic bytes (4 P in + 8 (11 + 3K) out per row) vs HBM peak;
  * device : load_ply_device(path) end to end (file in page cache, pinned
             double-buffered H2D + activation) -> wall seconds;
  * host   : load_ply_arrays(path) + DeviceScene.from_arrays (numpy / scipy
             activations on the host, then upload) -> wall seconds;
and prints one JSON line.  Usage: python tools/bench_ply.py [--n N] [--reps R]
"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=5_800_000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import ctypes

    import torch

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import _lib
    from paper_2409_08669_b200.projection import scene_struct
    from paper_2409_08669_b200.scene_io import PlySchema
    from ply_cases import write_ply

    n = args.n
    schema = PlySchema(3)
    names = list(schema.names)
    rng = np.random.default_rng(0)
    raw = rng.normal(0.0, 1.0, (n, len(names))).astype(np.float32)
    idx = {nm: i for i, nm in enumerate(names)}
    raw[:, idx["opacity"]] *= 3
    for c in ("scale_0", "scale_1", "scale_2"):
        raw[:, idx[c]] = rng.normal(-4.0, 1.0, n).astype(np.float32)
    out = {"metric": "ply_ingest", "n": n, "props": len(names)}
    with tempfile.TemporaryDirectory() as d:
        path = write_ply(Path(d) / "scene.ply", names, raw)
        out["file_bytes"] = path.stat().st_size
        # kernel alone
        P = len(names)
        draw = torch.from_numpy(raw).cuda()
        ds = ab.load_ply_device(path)          # warm-up + output allocation
        L = _lib.lib()
        status = torch.empty(2, dtype=torch.int64, device="cuda")
        st = torch.cuda.current_stream()
        cols = schema.device_columns(idx)
        cp = cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        sc = scene_struct(ds)
        times = []
        for _ in range(args.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            _lib.check(L.adr_ply_status_reset(_lib.ptr(status), st.cuda_stream))
            e0.record(st)
            _lib.check(L.adr_ply_activate(_lib.ptr(draw), 0, n, P, cp, ctypes.byref(sc), _lib.ptr(status),
                                          st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        k_ms = float(np.median(times[2:]))
        algo = n * (4 * P + 8 * (11 + 3 * schema.k))
        peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
            if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {}
        peak = float(peaks.get("hbm_gbs", 0) or 0) or None
        out["kernel"] = {"ms": round(k_ms, 4), "bytes": algo, "gbs": round(algo / k_ms / 1e6, 1),
                         "peak_gbs": peak, "frac": round(algo / k_ms / 1e6 / peak, 3) if peak else None}
        # end to end, device ingest
        dev_s = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            ds = ab.load_ply_device(path)
            torch.cuda.synchronize()
            dev_s.append(time.perf_counter() - t)
        out["device_e2e_s"] = round(float(np.median(dev_s)), 4)
        out["device_e2e_gbs_file"] = round(out["file_bytes"] / out["device_e2e_s"] / 1e9, 2)
        # host path
        t = time.perf_counter()
        arrays, deg = ab.load_ply_arrays(path)
        host = ab.DeviceScene.from_arrays(arrays, deg, "cuda", torch.float64)
        torch.cuda.synchronize()
        out["host_e2e_s"] = round(time.perf_counter() - t, 3)
        out["speedup_e2e"] = round(out["host_e2e_s"] / out["device_e2e_s"], 1)
        out["equal_to_host_path"] = all(torch.equal(getattr(ds, f), getattr(host, f))
                                        for f in ("centers", "scales", "rotations", "opacities", "sh"))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Digests of the REAL reference's load_ply (sb/scene.py:316-398) on the
deterministic checkpoints of tests/ply_cases.py, for the device-ingest parity
test (tests/test_gpu_ply.py).  Run in the build container, where
/root/reference exists:

    python tests/golden/make_ply_golden.py
"""
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

from ply_cases import CASES, write_case  # noqa: E402
from splatbench.scene import load_ply  # noqa: E402

FIELDS = ("centers", "scales", "rotations", "opacities", "sh")


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name in CASES:
            path = write_case(Path(d), name)
            with np.errstate(over="ignore"):
                arrays = load_ply(path).as_arrays()
            out[name] = {f: hashlib.sha256(np.ascontiguousarray(getattr(arrays, f), dtype=np.float64).tobytes()).hexdigest()
                         for f in FIELDS}
            out[name]["file_sha256"] = hashlib.sha256(path.read_bytes()).hexdigest()
            out[name]["n_inf_scales"] = int(np.isinf(arrays.scales).sum())
            out[name]["n_zero_scales"] = int((arrays.scales == 0).sum())
            print(name, out[name], flush=True)
    (HERE / "ply_digests.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

"""GPU: device-side PLY ingest (sb/scene.py:316-398 load_ply) through the
C-ABI (adr_ply_activate via scene_io.load_ply_device).

Parity is anchored on the reference itself, never on the box's own numpy
(whose float64 exp depends on the host CPU's SIMD dispatch):
  * the float64 exp / expit the kernel evaluates equal numpy's np.exp and
    scipy's expit on every float32 input (checksums made with numpy / scipy in
    the build container, tests/golden/exp64_exhaustive.json);
  * whole checkpoints load to the real splatbench's arrays
    (tests/golden/io_golden.npz, tests/golden/ply_digests.json).
"""
from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FIELDS = ("centers", "scales", "rotations", "opacities", "sh")


def _sha(t) -> str:
    return hashlib.sha256(np.ascontiguousarray(t.cpu().numpy(), dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("kind,name", [(0, "exp"), (1, "expit")])
def test_exp64_exhaustive_vs_numpy_scipy(kind, name):
    """exp_svml / expit_glibc == np.exp / scipy expit on all non-NaN float32
    inputs widened to float64, and on each named sub-range."""
    import torch

    from paper_2409_08669_b200 import _lib

    g = json.loads((GOLDEN / "exp64_exhaustive.json").read_text())
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = _lib.stream_handle(torch.cuda.current_stream())
    for rng_name, (lo, hi) in g["ranges"].items():
        _lib.check(_lib.lib().adr_exp64_checksum(kind, lo, hi, _lib.ptr(out), st))
        assert int(out.item()) % (1 << 64) == g[name][rng_name], rng_name


def test_device_ingest_equals_reference_golden():
    """io_scene_sh3.ply (40 Gaussians, SH 3) loads to splatbench's arrays."""
    import paper_2409_08669_b200 as ab

    with np.load(GOLDEN / "io_golden.npz") as z:
        want = {f: z[f"ply_{f}"] for f in FIELDS}
    ds = ab.load_ply_device(GOLDEN / "io_scene_sh3.ply")
    assert ds.sh_degree == 3 and len(ds) == 40
    for f in FIELDS:
        got = getattr(ds, f).cpu().numpy()
        assert got.dtype == np.float64
        assert np.array_equal(got.view(np.uint64), want[f].reshape(got.shape).view(np.uint64)), f


@pytest.mark.parametrize("name,chunk", [("sh3_extreme", 1 << 20), ("sh3_extreme", 32 << 20),
                                        ("sh0_shuffled", 4096), ("sh1_small", 1 << 20),
                                        ("sh2_reversed", 8192)])
def test_device_ingest_equals_reference_digests(name, chunk, tmp_path):
    """Extreme logits / log-scales across every exp and expit special case,
    shuffled / reversed / extra properties, many chunks: the device scene's
    bytes equal the real splatbench's arrays (tests/golden/ply_digests.json)."""
    import paper_2409_08669_b200 as ab
    from ply_cases import write_case

    want = json.loads((GOLDEN / "ply_digests.json").read_text())[name]
    path = write_case(tmp_path, name)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == want["file_sha256"]
    ds = ab.load_ply_device(path, chunk_bytes=chunk)
    for f in FIELDS:
        assert _sha(getattr(ds, f)) == want[f], f
    assert int(ds.scales.isinf().sum()) == want["n_inf_scales"]


def test_device_ingest_errors_match_reference(tmp_path):
    """First non-finite row (any property, checked before the quaternions),
    first zero-norm quaternion, header errors, empty file body."""
    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200.errors import SceneFormatError, SceneValidationError
    from ply_cases import make_raw, write_ply

    names, raw = make_raw("sh1_small")
    col = {nm: i for i, nm in enumerate(names)}
    bad = raw.copy()
    bad[300, col["nx"]] = np.nan
    bad[400, col["scale_1"]] = np.inf
    bad[[7, 350], col["rot_0"]] = 0.0
    for c in ("rot_1", "rot_2", "rot_3"):
        bad[[7, 350], col[c]] = 0.0
    p = write_ply(tmp_path / "a.ply", names, bad)
    with pytest.raises(SceneValidationError, match=r"non-finite value in element 300$"):
        ab.load_ply_device(p, chunk_bytes=4096)
    with pytest.raises(SceneValidationError, match=r"non-finite value in element 300$"):
        ab.load_ply_arrays(p)
    bad[300, col["nx"]] = 0.5
    bad[400, col["scale_1"]] = 0.5
    p = write_ply(tmp_path / "b.ply", names, bad)
    with pytest.raises(SceneValidationError, match=r"zero-norm quaternion in element 7$"):
        ab.load_ply_device(p, chunk_bytes=4096)
    with pytest.raises(SceneValidationError, match=r"zero-norm quaternion in element 7$"):
        ab.load_ply_arrays(p)
    (tmp_path / "c.ply").write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(SceneFormatError, match="binary_little_endian"):
        ab.load_ply_device(tmp_path / "c.ply")
    empty = write_ply(tmp_path / "d.ply", names, raw[:0])
    ds = ab.load_ply_device(empty)
    assert len(ds) == 0 and ds.sh.shape == (0, 4, 3)


def test_device_scene_from_file_uses_device_ingest(tmp_path):
    """DeviceScene.from_file on a PLY goes through adr_ply_activate (kernel
    launches counted by the library) and yields the reference's arrays."""
    import torch

    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import _lib

    before = _lib.lib().adr_kernel_launches()
    ds = ab.DeviceScene.from_file(GOLDEN / "io_scene_sh3.ply")
    assert _lib.lib().adr_kernel_launches() > before
    assert ds.centers.dtype == torch.float64
    with np.load(GOLDEN / "io_golden.npz") as z:
        for f in FIELDS:
            got = getattr(ds, f).cpu().numpy()
            assert np.array_equal(got.view(np.uint64), z[f"ply_{f}"].reshape(got.shape).view(np.uint64)), f

"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run on the B200 box
(`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_CASES = ("g_sh0_aabb", "g_sh3_baseline", "g_sh3_circle", "g_sh2_near_aabb", "g_sh1_small_aabb")
# edge semantics goldens (make_semantics_golden.py): term > 1, NaN term, NaN
# SH colours (chunked poisoning), extents beyond int32
SEMANTIC_CASES = ("g_term_gt1", "g_term_nan", "g_nan_sh", "g_huge_extent")
PROJ_FIELDS = ("valid", "mean2d", "cov2d", "conic", "depth", "color", "opacity", "lambda_max",
               "ext_x", "ext_y")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_camera(g: dict):
    from paper_2409_08669_b200 import Camera

    return Camera(view_matrix=g["cam_view_matrix"], fx=float(g["cam_fx"]), fy=float(g["cam_fy"]),
                  width=int(g["cam_width"]), height=int(g["cam_height"]),
                  near_plane=float(g["cam_near_plane"]),
                  background=tuple(float(v) for v in g["cam_background"]))


def golden_arrays(g: dict):
    from paper_2409_08669_b200 import SceneArrays

    return SceneArrays(g["centers"], g["scales"], g["rotations"], g["opacities"], g["sh"])


def config1_digests() -> dict:
    return json.loads((GOLDEN / "config1_digests.json").read_text())


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype.itemsize == b.dtype.itemsize and \
        np.array_equal(a.view(np.uint8), b.view(np.uint8))


def nan_bits_equal(a, b) -> bool:
    """Bit-exact, except that NaNs only need to be NaN in both (payloads of
    NaNs from NaN inputs are platform-specific)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype.itemsize != b.dtype.itemsize:
        return False
    if a.dtype.kind != "f":
        return np.array_equal(a.view(np.uint8), b.view(np.uint8))
    na, nb = np.isnan(a), np.isnan(b)
    u = np.uint32 if a.dtype.itemsize == 4 else np.uint64
    return bool(np.array_equal(na, nb) and np.array_equal(a.view(u)[~na], b.view(u)[~nb]))


def make_camera(width=64, height=64, distance=5.0, fov=60.0, background=(0.0, 0.0, 0.0)):
    """tests/conftest.py:9-13 of the reference."""
    from paper_2409_08669_b200 import Camera

    return Camera.from_lookat(position=(0.0, 0.0, -distance), target=(0.0, 0.0, 0.0),
                              fov_y_deg=fov, width=width, height=height, background=background)


def gaussian(center=(0, 0, 0), scale=(0.1, 0.1, 0.1), rotation=(1, 0, 0, 0), opacity=0.5,
             rgb=(1.0, 1.0, 1.0)):
    """Degree-0 Gaussian with colour ~rgb (reference tests/conftest.py:16-21)."""
    from paper_2409_08669_b200 import Gaussian3D

    dc = (np.asarray(rgb, dtype=np.float64) - 0.5) / 0.28209479177387814
    return Gaussian3D(center=center, scale=scale, rotation=rotation, opacity=opacity,
                      sh_coeffs=dc[None, :])


def make_scene(gs):
    from paper_2409_08669_b200 import Scene

    return Scene(gaussians=list(gs), sh_degree=0)


def mixed_spec():
    from paper_2409_08669_b200 import SyntheticSpec

    return SyntheticSpec(extent=1.2, scale_range=(0.01, 0.06), anisotropy_range=(1.0, 6.0),
                         opacity_range=(0.01, 1.0))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    orc.lib()
    return orc

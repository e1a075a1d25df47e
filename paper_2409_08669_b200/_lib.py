"""ctypes binding of libadrsplat.so (include/adr_splat.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from pathlib import Path

import numpy as np

from .errors import CapacityError, InternalError

_PKG = Path(__file__).resolve().parent
# ADR_LIBRARY overrides the in-tree build (used to A/B kernel variants: tools/variants.sh)
LIB_PATH = Path(os.environ.get("ADR_LIBRARY", _PKG / "_build" / "libadrsplat.so"))
CSRC = _PKG / "csrc"
HEADER = _PKG.parent / "include" / "adr_splat.h"

ADR_OK, ADR_ERR_VALUE, ADR_ERR_CAPACITY, ADR_ERR_INTERNAL, ADR_ERR_CUDA = range(5)
ADR_F32, ADR_F64 = 0, 1
MODE_CODES = {"baseline": 0, "circle": 1, "aabb": 2}

# Every symbol the header declares (checked by tests/test_capi_symbols.py).
EXPORTED = (
    "adr_abi_version", "adr_last_error", "adr_kernel_launches", "adr_device_sm_count", "adr_preprocess",
    "adr_touched_counts", "adr_inclusive_sum_scratch_bytes", "adr_inclusive_sum",
    "adr_duplicate_with_keys", "adr_sort_pairs_scratch_bytes", "adr_sort_pairs",
    "adr_identify_tile_ranges", "adr_render", "adr_exp_np_f32", "adr_selftest_exp", "adr_exp_checksum", "adr_exp64_checksum", "adr_render_selfcheck",
    "adr_ply_status_reset", "adr_ply_activate",
    "adr_frame_scratch_bytes", "adr_frame_record_offset", "adr_render_frame", "adr_preprocess_views", "adr_render_frame_post", "adr_image_loss_scratch_bytes", "adr_image_losses",
    "adr_render_reference_scratch_bytes", "adr_render_reference",
)


class Camera_t(ctypes.Structure):
    _fields_ = [("rot", ctypes.c_double * 9), ("trans", ctypes.c_double * 3),
                ("center", ctypes.c_double * 3), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("lim_x", ctypes.c_double), ("lim_y", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("background", ctypes.c_float * 3), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32)]


class Scene_t(ctypes.Structure):
    _fields_ = [("d_centers", ctypes.c_void_p), ("d_scales", ctypes.c_void_p),
                ("d_rotations", ctypes.c_void_p), ("d_opacities", ctypes.c_void_p),
                ("d_sh", ctypes.c_void_p), ("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32),
                ("dtype", ctypes.c_int32)]


class Projection_t(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in
                ("d_valid", "d_mean2d", "d_cov2d", "d_conic", "d_depth", "d_color", "d_opacity",
                 "d_lambda_max", "d_ext_x", "d_ext_y")]


class LoadStats_t(ctypes.Structure):
    _fields_ = [("sum", ctypes.c_int64), ("sum_sq", ctypes.c_int64), ("min", ctypes.c_int32),
                ("max", ctypes.c_int32)]


class FrameBuffers_t(ctypes.Structure):
    _fields_ = [("proj", Projection_t), ("d_pixels", ctypes.c_void_p), ("d_load", ctypes.c_void_p),
                ("d_keys", ctypes.c_void_p), ("d_gidx", ctypes.c_void_p),
                ("d_ranges", ctypes.c_void_p), ("d_counters", ctypes.c_void_p),
                ("d_stats", ctypes.c_void_p), ("d_hist", ctypes.c_void_p),
                ("hist_bins", ctypes.c_int32), ("d_scratch", ctypes.c_void_p),
                ("scratch_bytes", ctypes.c_size_t), ("pair_capacity", ctypes.c_int64),
                ("events", ctypes.c_void_p), ("projection_in_record", ctypes.c_int32)]


def build(verbose: bool = False) -> Path:
    """Compile libadrsplat.so in-tree (nvcc, sm_100a)."""
    cmd = ["make", "-C", str(CSRC), f"-j{min(8, os.cpu_count() or 1)}"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    """Load the library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the product path has no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        i32, i64, sz, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
        dbl = ctypes.c_double
        P = ctypes.POINTER
        sigs = {
            "adr_abi_version": (i32, []),
            "adr_last_error": (ctypes.c_char_p, []),
            "adr_kernel_launches": (i64, []),
            "adr_device_sm_count": (i32, []),
            "adr_preprocess": (i32, [P(Scene_t), P(Camera_t), i32, dbl, dbl, P(Projection_t), vp]),
            "adr_touched_counts": (i32, [P(Projection_t), i64, i32, i32, vp, vp]),
            "adr_inclusive_sum_scratch_bytes": (sz, [i64]),
            "adr_inclusive_sum": (i32, [vp, i64, vp, vp, vp, sz, vp]),
            "adr_duplicate_with_keys": (i32, [P(Projection_t), i64, vp, i32, i32, vp, vp, vp]),
            "adr_sort_pairs_scratch_bytes": (sz, [i64]),
            "adr_sort_pairs": (i32, [vp, vp, i64, i32, vp, vp, vp, sz, vp]),
            "adr_identify_tile_ranges": (i32, [vp, i64, i64, vp, vp, vp]),
            "adr_render": (i32, [P(Projection_t), i64, vp, i64, vp, P(Camera_t), dbl, dbl, vp, vp,
                                 vp, vp, i32, vp]),
            "adr_exp_np_f32": (i32, [vp, vp, i64, vp]),
            "adr_selftest_exp": (i32, [vp, vp]),
            "adr_render_selfcheck": (i32, [i32, vp]),
            "adr_exp_checksum": (i32, [ctypes.c_uint64, ctypes.c_uint64, vp, vp]),
            "adr_exp64_checksum": (i32, [i32, ctypes.c_uint64, ctypes.c_uint64, vp, vp]),
            "adr_ply_status_reset": (i32, [vp, vp]),
            "adr_ply_activate": (i32, [vp, i64, i64, i32, P(i32), P(Scene_t), vp, vp]),
            "adr_frame_scratch_bytes": (sz, [i64, i32, i32, i64]),
            "adr_frame_record_offset": (sz, [i64, i32, i32, i64]),
            "adr_render_frame": (i32, [P(Scene_t), P(Camera_t), i32, dbl, dbl, dbl,
                                       P(FrameBuffers_t), vp]),
            "adr_preprocess_views": (i32, [P(Scene_t), P(Camera_t), i32, i32, dbl, dbl,
                                           P(FrameBuffers_t), vp]),
            "adr_render_frame_post": (i32, [P(Scene_t), P(Camera_t), i32, dbl, dbl, dbl,
                                            P(FrameBuffers_t), vp]),
            "adr_image_loss_scratch_bytes": (sz, [i32, i32]),
            "adr_image_losses": (i32, [vp, vp, i32, i32, P(dbl), dbl, dbl, vp, vp, sz, vp]),
            "adr_render_reference_scratch_bytes": (sz, [i64]),
            "adr_render_reference": (i32, [P(Projection_t), i64, P(Camera_t), dbl, dbl, vp, vp, vp, sz, vp]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.adr_abi_version() != 3:
            raise RuntimeError("libadrsplat ABI mismatch")
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map an adr_status to the reference's exception types (sb/errors.py)."""
    if rc == ADR_OK:
        return
    msg = lib().adr_last_error().decode(errors="replace")
    if rc == ADR_ERR_VALUE:
        raise ValueError(msg)
    if rc == ADR_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == ADR_ERR_INTERNAL:
        raise InternalError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream) -> int:
    return int(stream.cuda_stream) if stream is not None else 0


def _fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def camera_struct(cam) -> Camera_t:
    """Camera constants with the reference's own expressions.

    ``center = -R.T @ t`` (sb/scene.py:158) is evaluated by numpy as the 3x3
    gemv FMA tree below (probed against numpy on 3000 random cameras);
    lim/cx/cy follow sb/projection.py:354-355,379-380 verbatim.
    """
    vm = np.asarray(cam.view_matrix, dtype=np.float64).reshape(4, 4)
    r = vm[:3, :3].tolist()
    t = vm[:3, 3].tolist()
    c = Camera_t()
    for i in range(3):
        for j in range(3):
            c.rot[3 * i + j] = r[i][j]
        c.trans[i] = t[i]
        c.center[i] = _fma(-r[2][i], t[2], _fma(-r[1][i], t[1], (-r[0][i]) * t[0]))
    c.fx, c.fy = float(cam.fx), float(cam.fy)
    c.lim_x = 1.3 * (0.5 * cam.width / cam.fx)
    c.lim_y = 1.3 * (0.5 * cam.height / cam.fy)
    c.cx = 0.5 * (cam.width - 1)
    c.cy = 0.5 * (cam.height - 1)
    c.near_plane = float(cam.near_plane)
    for i in range(3):
        c.background[i] = float(np.float32(cam.background[i]))
    c.width, c.height = int(cam.width), int(cam.height)
    return c

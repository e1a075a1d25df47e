"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module, and only as the checker or the
timed CPU baseline — never on the product path.

The functions mirror the reference stage functions one to one
(/root/reference/pkg/src/splatbench/, ``sb/`` below):

=========================  =================================
oracle function            reference
=========================  =================================
``camera_constants``       ``sb/projection.py:341-355``, ``sb/scene.py:147-158``
``preprocess``             ``sb/projection.py:291-420``
``touched_counts``         ``sb/tiling.py:77-114``
``inclusive_sum``          ``sb/tiling.py:117-122``
``duplicate_with_keys``    ``sb/tiling.py:125-156``
``sort_pairs``             ``sb/tiling.py:159-164``
``identify_tile_ranges``   ``sb/tiling.py:167-177``
``render``                 ``sb/render.py:57-171``
``run_pipeline``           ``sb/pipeline.py:85-124``
=========================  =================================
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"

MODES = {"baseline": 0, "circle": 1, "aabb": 2}
TILE_SIZE = 16


class _Camera(ctypes.Structure):
    _fields_ = [("rot", ctypes.c_double * 9), ("trans", ctypes.c_double * 3),
                ("center", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("lim_x", ctypes.c_double),
                ("lim_y", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("near_plane", ctypes.c_double), ("background", ctypes.c_float * 3),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


def build() -> Path:
    """Compile the oracle with its Makefile (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        _lib.orc_exp_np.restype = ctypes.c_float
        _lib.orc_exp_np.argtypes = [ctypes.c_float]
        _lib.orc_exp_checksum.restype = ctypes.c_uint64
        _lib.orc_exp_checksum.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        for fn in ("orc_exp_svml", "orc_exp_glibc", "orc_expit"):
            getattr(_lib, fn).restype = ctypes.c_double
            getattr(_lib, fn).argtypes = [ctypes.c_double]
        _lib.orc_exp64_checksum.restype = ctypes.c_uint64
        _lib.orc_exp64_checksum.argtypes = [ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64]
        _lib.orc_log.restype = ctypes.c_double
        _lib.orc_log.argtypes = [ctypes.c_double]
        _lib.orc_inclusive_sum.restype = ctypes.c_int32
        _lib.orc_identify_tile_ranges.restype = ctypes.c_int32
        _lib.orc_ceil_ambiguous.restype = ctypes.c_int32
        _lib.orc_ceil_ambiguous.argtypes = [ctypes.c_double, ctypes.c_double]
        _lib.orc_preprocess_ambiguous.restype = ctypes.c_int64
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def _fma(a: float, b: float, c: float) -> float:
    """Exactly rounded fused multiply-add on Python floats."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def camera_constants(cam) -> _Camera:
    """Host constants for one camera.

    ``center`` is ``-R.T @ t`` (sb/scene.py:158); numpy evaluates that 3x3
    gemv as the FMA tree below (probed: equal on 3000 random cameras).
    """
    vm = np.asarray(cam.view_matrix, dtype=np.float64).reshape(4, 4)
    r = vm[:3, :3].tolist()
    t = vm[:3, 3].tolist()
    c = _Camera()
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


@dataclass
class SceneArrays:
    centers: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray
    sh_degree: int

    def __len__(self):
        return len(self.opacities)


def scene_arrays(scene) -> SceneArrays:
    """fp64 contiguous arrays from a reference Scene, a SceneArrays, or a dict."""
    if isinstance(scene, SceneArrays):
        return scene
    if isinstance(scene, dict):
        d = scene
        deg = int(d["sh_degree"])
    elif hasattr(scene, "as_arrays"):
        a = scene.as_arrays()
        d = {"centers": a.centers, "scales": a.scales, "rotations": a.rotations,
             "opacities": a.opacities, "sh": a.sh}
        deg = int(scene.sh_degree)
    else:
        d = {k: np.asarray(getattr(scene, k)) for k in
             ("centers", "scales", "rotations", "opacities", "sh")}
        deg = int(scene.sh_degree)
    k = (deg + 1) ** 2
    f = lambda x, shape: np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(shape))
    n = len(np.asarray(d["opacities"]).reshape(-1))
    return SceneArrays(f(d["centers"], (n, 3)), f(d["scales"], (n, 3)), f(d["rotations"], (n, 4)),
                       f(d["opacities"], (n,)), f(d["sh"], (n, k, 3)), deg)


def exp_np(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    f = lib().orc_exp_np
    for i, v in enumerate(x.ravel().tolist()):
        out.flat[i] = f(v)
    return out


def preprocess(scene, cam, mode="aabb", alpha_low=1.0 / 255.0, dilation=0.3, threads=0):
    if not 0.0 < alpha_low < 1.0:
        raise ValueError("alpha_low must lie in (0, 1)")
    if dilation < 0:
        raise ValueError("dilation must be non-negative")
    mode = getattr(mode, "value", mode)
    s = scene_arrays(scene)
    n = len(s)
    out = {
        "valid": np.zeros(n, dtype=np.bool_),
        "mean2d": np.zeros((n, 2), dtype=np.float32),
        "cov2d": np.zeros((n, 3), dtype=np.float32),
        "conic": np.zeros((n, 3), dtype=np.float32),
        "depth": np.zeros(n, dtype=np.float32),
        "color": np.zeros((n, 3), dtype=np.float32),
        "opacity": np.zeros(n, dtype=np.float32),
        "lambda_max": np.zeros(n, dtype=np.float32),
        "ext_x": np.zeros(n, dtype=np.int32),
        "ext_y": np.zeros(n, dtype=np.int32),
    }
    if n:
        c = camera_constants(cam)
        lib().orc_preprocess(
            ctypes.c_int64(n), ctypes.c_int32(s.sh_degree), _p(s.centers), _p(s.scales),
            _p(s.rotations), _p(s.opacities), _p(s.sh), ctypes.byref(c),
            ctypes.c_int32(MODES[mode]), ctypes.c_double(alpha_low), ctypes.c_double(dilation),
            _p(out["valid"]), _p(out["mean2d"]), _p(out["cov2d"]), _p(out["conic"]),
            _p(out["depth"]), _p(out["color"]), _p(out["opacity"]), _p(out["lambda_max"]),
            _p(out["ext_x"]), _p(out["ext_y"]), ctypes.c_int32(threads or os.cpu_count()))
    # extents whose ceil could flip under a 2-ulp change of the fp64 log
    # (orc_ceil_ambiguous): 0 proves numpy's log gives the same extents
    out["ambiguous_extents"] = int(lib().orc_preprocess_ambiguous()) if n else 0
    return out


def grid_dims(width, height):
    return -(-width // TILE_SIZE), -(-height // TILE_SIZE)


def touched_counts(proj, width, height):
    tx, ty = grid_dims(width, height)
    n = len(proj["valid"])
    counts = np.zeros(n, dtype=np.int64)
    if n:
        lib().orc_touched_counts(ctypes.c_int64(n), _p(proj["mean2d"]), _p(proj["ext_x"]),
                                 _p(proj["ext_y"]), _p(proj["valid"].view(np.uint8)),
                                 ctypes.c_int32(tx), ctypes.c_int32(ty), _p(counts))
    return counts


def inclusive_sum(counts):
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    out = np.zeros(len(counts), dtype=np.int64)
    if len(counts) and lib().orc_inclusive_sum(ctypes.c_int64(len(counts)), _p(counts), _p(out)):
        raise OverflowError("pair count overflows the 64-bit index type")
    return out


def duplicate_with_keys(proj, offsets, width, height):
    tx, ty = grid_dims(width, height)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    total = int(offsets[-1]) if len(offsets) else 0
    keys = np.empty(total, dtype=np.uint64)
    gidx = np.empty(total, dtype=np.int64)
    if total:
        lib().orc_duplicate_with_keys(
            ctypes.c_int64(len(offsets)), _p(proj["mean2d"]), _p(proj["ext_x"]),
            _p(proj["ext_y"]), _p(proj["valid"].view(np.uint8)), _p(proj["depth"]),
            _p(offsets), ctypes.c_int32(tx), ctypes.c_int32(ty), _p(keys), _p(gidx))
    return keys, gidx


def sort_pairs(keys, gidx):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    gidx = np.ascontiguousarray(gidx, dtype=np.int64)
    ko, go = np.empty_like(keys), np.empty_like(gidx)
    if len(keys):
        lib().orc_sort_pairs(ctypes.c_int64(len(keys)), _p(keys), _p(gidx), _p(ko), _p(go))
    return ko, go


def identify_tile_ranges(sorted_keys, n_tiles):
    sorted_keys = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
    ranges = np.zeros((n_tiles, 2), dtype=np.int64)
    rc = lib().orc_identify_tile_ranges(ctypes.c_int64(len(sorted_keys)), _p(sorted_keys),
                                        ctypes.c_int64(n_tiles), _p(ranges))
    if rc:
        raise RuntimeError("keys are not sorted" if rc == 1 else
                           "key references a tile outside the grid")
    return ranges


def render(proj, gidx, ranges, cam, alpha_low=1.0 / 255.0, term_threshold=1e-4, threads=0,
           tile_stride=1, tile_phase=0):
    w, h = int(cam.width), int(cam.height)
    tx, ty = grid_dims(w, h)
    pixels = np.zeros((h, w, 3), dtype=np.float32)
    counts = np.zeros((h, w), dtype=np.int32)
    bg = np.asarray(cam.background, dtype=np.float32)
    gidx = np.ascontiguousarray(gidx, dtype=np.int64)
    ranges = np.ascontiguousarray(ranges, dtype=np.int64)
    lib().orc_render(ctypes.c_int32(w), ctypes.c_int32(h), ctypes.c_int32(tx), ctypes.c_int32(ty),
                     _p(proj["mean2d"]), _p(proj["conic"]), _p(proj["opacity"]),
                     _p(proj["color"]), _p(gidx), _p(ranges), _p(bg),
                     ctypes.c_double(alpha_low), ctypes.c_double(term_threshold), _p(pixels),
                     _p(counts), ctypes.c_int32(tile_stride), ctypes.c_int32(tile_phase),
                     ctypes.c_int32(threads or os.cpu_count()))
    return pixels, counts


def run_pipeline(scene, cam, mode="aabb", alpha_low=1.0 / 255.0, threads=0, dilation=0.3,
                 term_threshold=1e-4, tile_stride=1):
    """All six stages; returns a dict with every intermediate and stage times.

    ``tile_stride > 1`` renders only every ``tile_stride``-th tile (the bounded
    CPU-baseline sample of bench.py); everything else is the full frame.
    """
    w, h = int(cam.width), int(cam.height)
    tx, ty = grid_dims(w, h)
    t0 = time.perf_counter()
    proj = preprocess(scene, cam, mode, alpha_low, dilation, threads)
    t1 = time.perf_counter()
    counts = touched_counts(proj, w, h)
    offsets = inclusive_sum(counts)
    t2 = time.perf_counter()
    keys, gidx = duplicate_with_keys(proj, offsets, w, h)
    t3 = time.perf_counter()
    skeys, sgidx = sort_pairs(keys, gidx)
    t4 = time.perf_counter()
    ranges = identify_tile_ranges(skeys, tx * ty)
    t5 = time.perf_counter()
    pixels, load = render(proj, sgidx, ranges, cam, alpha_low, term_threshold, threads,
                          tile_stride=tile_stride)
    t6 = time.perf_counter()
    return {"projection": proj, "counts": counts, "offsets": offsets, "keys_unsorted": keys,
            "gidx_unsorted": gidx, "keys": skeys, "gidx": sgidx, "ranges": ranges,
            "pixels": pixels, "load": load,
            "times": {"preprocess": t1 - t0, "inclusivesum": t2 - t1, "duplicate": t3 - t2,
                      "sort": t4 - t3, "ranges": t5 - t4, "render": t6 - t5}}

"""ctypes loader for librade.so (the C ABI declared in include/rade.h).

There is no fallback: if the library is missing or fails to load this raises, loudly.
Build it with `python -m paper_2406_01467_b200.build` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RADE_LIB selects another build of the same ABI (e.g. librade_checks.so, the RD_CHECKS build)
LIB_PATH = os.environ.get("RADE_LIB") or os.path.join(HERE, "librade.so")

RD_OK, RD_ERR_INVALID_ARGUMENT, RD_ERR_STATE, RD_ERR_ALLOC, RD_ERR_CUDA = range(5)
STATUS_NAMES = {0: "RD_OK", 1: "RD_ERR_INVALID_ARGUMENT", 2: "RD_ERR_STATE", 3: "RD_ERR_ALLOC", 4: "RD_ERR_CUDA"}


class RadeError(RuntimeError):
    def __init__(self, status, func, msg):
        super().__init__(f"{func} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class RdCamera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("R", ctypes.c_float * 9),
                ("t", ctypes.c_float * 3), ("znear", ctypes.c_float)]


class RdOptions(ctypes.Structure):
    _fields_ = [("tile", ctypes.c_int32), ("alpha_min", ctypes.c_float), ("alpha_max", ctypes.c_float),
                ("T_min", ctypes.c_float), ("median_T", ctypes.c_float), ("dilation", ctypes.c_float),
                ("bg", ctypes.c_float * 3), ("sh_degree", ctypes.c_int32), ("guard_band", ctypes.c_float)]


class RdGaussians(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_coeffs", ctypes.c_int32), ("means", ctypes.c_void_p),
                ("scales", ctypes.c_void_p), ("rotations", ctypes.c_void_p), ("opacities", ctypes.c_void_p),
                ("sh", ctypes.c_void_p), ("filter3d", ctypes.c_void_p)]


class RdGrads(ctypes.Structure):
    _fields_ = [("means", ctypes.c_void_p), ("scales", ctypes.c_void_p), ("rotations", ctypes.c_void_p),
                ("opacities", ctypes.c_void_p), ("sh", ctypes.c_void_p), ("means2d", ctypes.c_void_p)]


class RdTsdf(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_float * 3), ("voxel_size", ctypes.c_float), ("dims", ctypes.c_int32 * 3),
                ("truncation", ctypes.c_float), ("max_depth", ctypes.c_float), ("tsdf", ctypes.c_void_p),
                ("weight", ctypes.c_void_p)]


class RdFwdMaps(ctypes.Structure):
    _fields_ = [("color", ctypes.c_void_p), ("depth", ctypes.c_void_p), ("normal", ctypes.c_void_p),
                ("alpha", ctypes.c_void_p), ("distortion", ctypes.c_void_p)]


class RdBwdCotangents(ctypes.Structure):
    _fields_ = [("dL_dcolor", ctypes.c_void_p), ("dL_ddepth", ctypes.c_void_p), ("dL_dnormal", ctypes.c_void_p),
                ("dL_dalpha", ctypes.c_void_p), ("dL_ddistortion", ctypes.c_void_p)]


class RdStats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_duplicates", ctypes.c_int64), ("tiles_x", ctypes.c_int32),
                ("tiles_y", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("stage", ctypes.c_int32), ("key_bits", ctypes.c_int32), ("n_visible", ctypes.c_int64),
                ("n_big", ctypes.c_int64)]


RD_NUM_KERNELS = 9
KERNEL_NAMES = ["preprocess_fwd", "depth_sort", "scan", "duplicate", "tile_sort", "ranges", "render_fwd", "render_bwd",
                "preprocess_bwd"]


class RdTimings(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * RD_NUM_KERNELS), ("launches", ctypes.c_int64 * RD_NUM_KERNELS),
                ("pairs_evaluated_fwd", ctypes.c_int64), ("pairs_blended_fwd", ctypes.c_int64),
                ("pairs_evaluated_bwd", ctypes.c_int64), ("n_visible", ctypes.c_int64),
                ("n_duplicates", ctypes.c_int64), ("views", ctypes.c_int64), ("n_visible_union", ctypes.c_int64),
                ("n_culled", ctypes.c_int64 * 6), ("pairs_issued_fwd", ctypes.c_int64)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)

# exported symbols and their signatures (every function declared in include/rade.h)
_VP = ctypes.c_void_p
SIGNATURES = {
    "rd_options_default": ([ctypes.POINTER(RdOptions)], ctypes.c_int),
    "rd_view_create": ([ctypes.POINTER(_VP), ALLOC_FN, FREE_FN, _VP], ctypes.c_int),
    "rd_view_destroy": ([_VP], ctypes.c_int),
    "rd_preprocess": ([_VP, ctypes.POINTER(RdGaussians), ctypes.POINTER(RdCamera), ctypes.POINTER(RdOptions), _VP],
                      ctypes.c_int),
    "rd_bin": ([_VP, ctypes.POINTER(ctypes.c_int64), _VP], ctypes.c_int),
    "rd_render_fwd": ([_VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_render_bwd": ([_VP, ctypes.POINTER(RdGaussians), _VP, _VP, _VP, _VP, ctypes.POINTER(RdGrads), _VP],
                      ctypes.c_int),
    "rd_blend_bwd": ([_VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_render_fwd_ex": ([_VP, ctypes.POINTER(RdFwdMaps), _VP], ctypes.c_int),
    "rd_normal_consistency": ([ctypes.POINTER(RdCamera), _VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_tsdf_integrate": ([ctypes.POINTER(RdTsdf), _VP, ctypes.POINTER(RdCamera), ctypes.c_int32, _VP], ctypes.c_int),
    "rd_marching_cubes": ([ctypes.POINTER(RdTsdf), ctypes.c_float, _VP, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                           _VP], ctypes.c_int),
    "rd_normal_consistency_bwd": ([ctypes.POINTER(RdCamera), _VP, _VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_blend_bwd_ex": ([_VP, ctypes.POINTER(RdBwdCotangents), _VP], ctypes.c_int),
    "rd_preprocess_bwd": ([_VP, ctypes.POINTER(RdGaussians), ctypes.POINTER(RdGrads), _VP], ctypes.c_int),
    "rd_preprocess_bwd_views": ([ctypes.POINTER(_VP), ctypes.c_int32, ctypes.POINTER(RdGaussians),
                                 ctypes.POINTER(RdGrads), _VP], ctypes.c_int),
    "rd_preprocess_bwd_geometry": ([_VP, ctypes.POINTER(RdGaussians), ctypes.POINTER(RdGrads), _VP], ctypes.c_int),
    "rd_preprocess_bwd_views_sh": ([ctypes.POINTER(_VP), ctypes.c_int32, ctypes.POINTER(RdGaussians),
                                    ctypes.POINTER(RdGrads), _VP], ctypes.c_int),
    "rd_preprocess_views": ([ctypes.POINTER(_VP), ctypes.c_int32, ctypes.POINTER(RdGaussians),
                             ctypes.POINTER(RdCamera), ctypes.POINTER(RdOptions), _VP], ctypes.c_int),
    "rd_preprocess_bwd_views_ex": ([ctypes.POINTER(_VP), ctypes.c_int32, ctypes.POINTER(RdGaussians),
                                    ctypes.POINTER(RdGrads), ctypes.c_uint32, _VP], ctypes.c_int),
    "rd_view_stats": ([_VP, ctypes.POINTER(RdStats)], ctypes.c_int),
    "rd_set_profiling": ([_VP, ctypes.c_int32], ctypes.c_int),
    "rd_get_timings": ([_VP, ctypes.POINTER(RdTimings), ctypes.c_int32], ctypes.c_int),
    "rd_debug_binning": ([_VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_debug_preprocess": ([_VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_debug_pixel_state": ([_VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "rd_debug_grads2d": ([_VP, _VP, _VP], ctypes.c_int),
    "rd_last_error": ([], ctypes.c_char_p),
    "rd_version": ([], ctypes.c_char_p),
}

_lib = None


def load(path: str = LIB_PATH):
    """Loads librade.so and binds every symbol of include/rade.h. Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: the CUDA extension is not built "
                          f"(run `python -m paper_2406_01467_b200.build`). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(status: int, func: str):
    if status != RD_OK:
        msg = load().rd_last_error()
        raise RadeError(status, func, msg.decode() if msg else "")

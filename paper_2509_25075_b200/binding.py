"""ctypes marshalling for libgem.so (include/gem.h).  Argument marshalling only:
every step of the GEM path runs in the library's CUDA kernels.  There is no
CPU fallback — if libgem.so is missing or fails to load this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgem.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "gem.h")

GEM_OK, GEM_E_INVALID, GEM_E_SHAPE, GEM_E_ALIGN, GEM_E_CUDA, GEM_E_CUFFT, GEM_E_CAPACITY, GEM_E_STATE, \
    GEM_E_NONFINITE = range(9)
GEM_MEM_DEVICE, GEM_MEM_HOST = 0, 1
GEM_FLAG_FUSED = 1
GEM_FLAG_NO_ROTATION = 2   # Table 5 ablation: R fixed to I
GEM_FLAG_ISOTROPIC = 4     # Table 5 ablation: tied log-scales
GEM_FLAG_ZSORT = 8         # P:227 z-sorted per-tile lists
GEM_FLAG_ELLIPSE = 16      # per-pixel: inside the k-sigma ellipse
GEM_FLAG_PIXEL_TAU = 32    # per-pixel: |G| >= tau (Eq. 8)
GEM_FLAG_EXACT_TILES = 64  # lists: only tiles holding a kept pixel


class GemConfigC(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int32), ("pixel_size", ctypes.c_float), ("n_gauss", ctypes.c_int64),
                ("max_batch", ctypes.c_int32), ("cull_k", ctypes.c_float), ("tau", ctypes.c_float),
                ("tile", ctypes.c_int32), ("list_capacity", ctypes.c_int64),
                ("lr_mean", ctypes.c_float), ("lr_log_scale", ctypes.c_float), ("lr_quat", ctypes.c_float),
                ("lr_density", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("flags", ctypes.c_uint32), ("wave", ctypes.c_int32)]


class GemSoaC(ctypes.Structure):
    _fields_ = [("mean_rho", ctypes.c_void_p), ("log_scale", ctypes.c_void_p), ("quat", ctypes.c_void_p)]


class GemBatchC(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("memory", ctypes.c_int32), ("rot", ctypes.c_void_p),
                ("shift", ctypes.c_void_p), ("ctf", ctypes.c_void_p), ("observed", ctypes.c_void_p)]


class GemStatsC(ctypes.Structure):
    _fields_ = [("entries", ctypes.c_int64), ("capacity", ctypes.c_int64), ("degenerate", ctypes.c_int32),
                ("overflow", ctypes.c_int32), ("nonfinite", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("pairs", ctypes.c_int64), ("wave", ctypes.c_int32),
                ("fused", ctypes.c_int32)]


class GemKernelTimeC(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("launches", ctypes.c_int32), ("total_ms", ctypes.c_double)]


class GemError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


def header_symbols():
    """Names of every function include/gem.h declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"GEM_API\s+[\w\s\*]+?\b(gem_\w+)\s*\(", txt)))


_lib = None


def lib():
    """Load libgem.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built — run `python -m paper_2509_25075_b200.build` "
                           "(__graft_entry__.build()); the GEM step has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    p, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    L.gem_workspace_bytes.restype = sz
    L.gem_workspace_bytes.argtypes = [ctypes.POINTER(GemConfigC)]
    L.gem_init.restype = ctypes.c_int
    L.gem_init.argtypes = [ctypes.POINTER(GemConfigC), p, sz, p, ctypes.POINTER(p)]
    L.gem_destroy.restype = ctypes.c_int
    L.gem_destroy.argtypes = [p]
    L.gem_forward.restype = ctypes.c_int
    L.gem_forward.argtypes = [p, ctypes.POINTER(GemSoaC), ctypes.POINTER(GemBatchC), p, p, p, p]
    L.gem_backward.restype = ctypes.c_int
    L.gem_backward.argtypes = [p, ctypes.POINTER(GemSoaC), ctypes.POINTER(GemSoaC), p]
    L.gem_step.restype = ctypes.c_int
    L.gem_step.argtypes = [p, ctypes.POINTER(GemSoaC), ctypes.POINTER(GemSoaC), ctypes.POINTER(GemSoaC),
                           ctypes.POINTER(GemSoaC), i64, p]
    L.gem_render_volume.restype = ctypes.c_int
    L.gem_render_volume.argtypes = [p, ctypes.POINTER(GemSoaC), i32, ctypes.c_float, p, p, sz, p]
    L.gem_volume_scratch_bytes.restype = sz
    L.gem_volume_scratch_bytes.argtypes = [p, i32, ctypes.c_float]
    L.gem_export_lists.restype = ctypes.c_int
    L.gem_export_lists.argtypes = [p, i32, p, p, i64, p]
    L.gem_stats.restype = ctypes.c_int
    L.gem_stats.argtypes = [p, ctypes.POINTER(GemStatsC)]
    L.gem_profile_enable.restype = ctypes.c_int
    L.gem_profile_enable.argtypes = [p, i32]
    L.gem_profile_read.restype = i32
    L.gem_profile_read.argtypes = [p, ctypes.POINTER(GemKernelTimeC), i32]
    L.gem_last_launch_count.restype = i32
    L.gem_last_launch_count.argtypes = [p]
    L.gem_status_string.restype = ctypes.c_char_p
    L.gem_status_string.argtypes = [ctypes.c_int]
    _lib = L
    return L


def status_string(s):
    try:
        return lib().gem_status_string(int(s)).decode()
    except Exception:  # library unavailable
        return str(s)


def check(status, where):
    if status != GEM_OK:
        raise GemError(status, where)

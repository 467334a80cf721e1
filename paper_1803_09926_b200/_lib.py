"""ctypes loader for the in-tree ``libdwconv.so`` (include/dwconv.h).

Argument marshalling only.  There is no CPU fallback: if the library is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdwconv.so")

NCHW, NHWC = 0, 1
F32, BF16 = 0, 1
PASS_FWD, PASS_BWD_DATA, PASS_BWD_FILTER, PASS_BWD = 0, 1, 2, 3
VARIANTS = {0: "none", 1: "generic", 2: "nchw_chunk", 3: "nhwc_tile", 4: "nhwc_tma", 5: "nhwc_bdmma", 6: "nhwc_gen"}
FUNCTIONS = ("dwconv_abi_version", "dwconv_status_string", "dwconv_output_shape", "dwconv_fwd",
             "dwconv_bwd_data", "dwconv_bwd_filter_workspace_bytes", "dwconv_bwd_filter",
             "dwconv_bwd_workspace_bytes", "dwconv_bwd",
             "dwconv_workspace_init", "dwconv_plan", "dwconv_plan_candidates", "dwconv_plan_select",
             "dwconv_set_variant_override", "dwconv_plan_create", "dwconv_plan_destroy", "dwconv_plan_describe",
             "dwconv_plan_workspace_bytes", "dwconv_fwd_plan", "dwconv_bwd_data_plan", "dwconv_bwd_filter_plan",
             "dwconv_bwd_plan")
MAX_CANDIDATES = 48


class Desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("c", ctypes.c_int64), ("h", ctypes.c_int64), ("w", ctypes.c_int64),
                ("multiplier", ctypes.c_int32), ("kh", ctypes.c_int32), ("kw", ctypes.c_int32),
                ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32),
                ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("dtype", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("grid", ctypes.c_int32), ("block", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("launches", ctypes.c_int32), ("work_units", ctypes.c_int64),
                ("planes_per_chunk", ctypes.c_int32), ("rows_per_band", ctypes.c_int32),
                ("batch_slices", ctypes.c_int32), ("max_chain", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("kernel_family", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class DwconvError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_1803_09926_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    dp = ctypes.POINTER(Desc)
    lib.dwconv_abi_version.restype = i32
    lib.dwconv_status_string.argtypes = [i32]
    lib.dwconv_status_string.restype = ctypes.c_char_p
    lib.dwconv_output_shape.argtypes = [dp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.dwconv_fwd.argtypes = [dp, vp, vp, vp, vp]
    lib.dwconv_bwd_data.argtypes = [dp, vp, vp, vp, vp]
    lib.dwconv_bwd_filter_workspace_bytes.argtypes = [dp]
    lib.dwconv_bwd_filter_workspace_bytes.restype = sz
    lib.dwconv_bwd_filter.argtypes = [dp, vp, vp, vp, vp, sz, vp]
    lib.dwconv_bwd_workspace_bytes.argtypes = [dp]
    lib.dwconv_bwd_workspace_bytes.restype = sz
    lib.dwconv_bwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.dwconv_workspace_init.argtypes = [vp, sz, vp]
    lib.dwconv_plan.argtypes = [dp, i32, ctypes.POINTER(PlanInfo)]
    lib.dwconv_plan_candidates.argtypes = [dp, i32, i32, ctypes.POINTER(PlanInfo), ctypes.POINTER(i32)]
    lib.dwconv_plan_select.argtypes = [dp, i32, i32]
    lib.dwconv_set_variant_override.argtypes = [i32]
    lib.dwconv_plan_create.argtypes = [dp, i32, i32, ctypes.POINTER(vp)]
    lib.dwconv_plan_destroy.argtypes = [vp]
    lib.dwconv_plan_destroy.restype = None
    lib.dwconv_plan_describe.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.dwconv_plan_workspace_bytes.argtypes = [vp]
    lib.dwconv_plan_workspace_bytes.restype = sz
    lib.dwconv_fwd_plan.argtypes = [vp, vp, vp, vp, vp]
    lib.dwconv_bwd_data_plan.argtypes = [vp, vp, vp, vp, vp]
    lib.dwconv_bwd_filter_plan.argtypes = [vp, vp, vp, vp, vp, sz, vp]
    lib.dwconv_bwd_plan.argtypes = [vp, vp, vp, vp, vp, vp, vp, sz, vp]
    for f in ("dwconv_plan_create", "dwconv_plan_describe", "dwconv_fwd_plan", "dwconv_bwd_data_plan",
              "dwconv_bwd_filter_plan", "dwconv_bwd_plan"):
        getattr(lib, f).restype = i32
    for f in ("dwconv_output_shape", "dwconv_fwd", "dwconv_bwd_data", "dwconv_bwd_filter", "dwconv_bwd",
              "dwconv_workspace_init", "dwconv_plan", "dwconv_plan_candidates", "dwconv_plan_select",
              "dwconv_set_variant_override"):
        getattr(lib, f).restype = i32
    if lib.dwconv_abi_version() != 2:
        raise RuntimeError("libdwconv ABI version mismatch")
    _lib = lib
    return lib


def status_string(status: int) -> str:
    return load().dwconv_status_string(status).decode()


def check(status: int, where: str) -> None:
    if status != 0:
        raise DwconvError(status, where)

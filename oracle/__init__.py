"""CPU oracle for the depthwise-convolution training layer -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1803_09926_b200``) never imports it and shares no code
with it: the arithmetic lives in ``oracle/dw_oracle.c`` (plain C, double
precision, nested loops; see its header for the paper passages each function
follows), and this module only marshals numpy arrays into it.

Parity status of each function (DESIGN.md §4 lists the pins):
  fwd, bwd_data, bwd_filter    pinned: P1-P8 in tests/test_oracle.py
  their sum|terms| outputs     pinned: P7b (torch CPU fp64 conv2d / conv2d_input /
                               conv2d_weight of |x|, |w|, |dy|: bitwise on integers)
  dense_* / expand / mask      pinned: P7 (torch CPU fp64 conv2d), P1/P2
  round (storage rounding)     pinned: numpy fp32 casts, hand-built bf16 cases
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
NCHW, NHWC = 0, 1
F32, BF16 = 0, 1

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fopenmp",
                               "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64, i32 = ctypes.c_int64, ctypes.c_int
        dw_args = [dp, dp, dp, dp, i64, i64, i64, i64, i32, i32, i32, i32, i32, i32, i32, i32]
        for name in ("oracle_dw_fwd", "oracle_dw_bwd_data", "oracle_dw_bwd_filter"):
            getattr(lib, name).argtypes = dw_args
            getattr(lib, name).restype = None
        dense_args = [dp, dp, dp, i64, i64, i64, i64, i64, i32, i32, i32, i32, i32, i32]
        for name in ("oracle_dense_fwd", "oracle_dense_bwd_data", "oracle_dense_bwd_filter"):
            getattr(lib, name).argtypes = dense_args
            getattr(lib, name).restype = None
        lib.oracle_expand_weights.argtypes = [dp, dp, i64, i32, i32, i32]
        lib.oracle_mask.argtypes = [dp, i64, i32, i32, i32]
        lib.oracle_hadamard.argtypes = [dp, dp, dp, i64]
        lib.oracle_round.argtypes = [dp, dp, i64, i32]
        lib.oracle_out_size.argtypes = [i64, i32, i32, i32, ctypes.POINTER(i64)]
        lib.oracle_out_size.restype = i32
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_set_threads.restype = None
        lib.oracle_get_threads.argtypes = []
        lib.oracle_get_threads.restype = i32
        _lib = lib
    return _lib


def set_threads(t: int) -> None:
    """Outer-loop OpenMP threads for fwd / bwd_data / bwd_filter (1 = sequential, the default).  Every
    output element is still summed by one thread in definition order: results are bitwise unchanged."""
    _load().oracle_set_threads(int(t))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def out_size(n: int, k: int, s: int, p: int) -> Optional[int]:
    o = ctypes.c_int64()
    ok = _load().oracle_out_size(n, k, s, p, ctypes.byref(o))
    return int(o.value) if ok else None


def _shape_args(xshape, layout):
    if layout == NCHW:
        N, C, H, W = xshape
    else:
        N, H, W, C = xshape
    return N, C, H, W


def _act_shape(N, C, H, W, layout):
    return (N, C, H, W) if layout == NCHW else (N, H, W, C)


def _hw(k, s, p):
    k = (k, k) if np.isscalar(k) else tuple(k)
    s = (s, s) if np.isscalar(s) else tuple(s)
    p = (p, p) if np.isscalar(p) else tuple(p)
    return k, s, p


def fwd(x, w, stride=1, padding=0, layout=NCHW) -> Tuple[np.ndarray, np.ndarray]:
    """y (unrounded double) and per-element sum|terms|.  w: [C*m, kh, kw]."""
    x, w = _d(x), _d(w)
    N, C, H, W = _shape_args(x.shape, layout)
    Co, kh, kw = w.shape[0], w.shape[-2], w.shape[-1]
    m = Co // C
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    Ho, Wo = out_size(H, kh, sh, ph), out_size(W, kw, sw, pw)
    if Ho is None or Wo is None or Ho < 1 or Wo < 1:
        raise ValueError("kernel exceeds padded input")
    y = np.zeros(_act_shape(N, Co, Ho, Wo, layout))
    a = np.zeros_like(y)
    _load().oracle_dw_fwd(_p(x), _p(w), _p(y), _p(a), N, C, H, W, m, kh, kw, sh, sw, ph, pw, layout)
    return y, a


def bwd_data(dy, w, xshape, stride=1, padding=0, layout=NCHW) -> Tuple[np.ndarray, np.ndarray]:
    dy, w = _d(dy), _d(w)
    N, C, H, W = _shape_args(xshape, layout)
    Co, kh, kw = w.shape[0], w.shape[-2], w.shape[-1]
    m = Co // C
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    dx = np.zeros(_act_shape(N, C, H, W, layout))
    a = np.zeros_like(dx)
    _load().oracle_dw_bwd_data(_p(dy), _p(w), _p(dx), _p(a), N, C, H, W, m, kh, kw, sh, sw, ph, pw, layout)
    return dx, a


def bwd_filter(x, dy, wshape, stride=1, padding=0, layout=NCHW) -> Tuple[np.ndarray, np.ndarray]:
    x, dy = _d(x), _d(dy)
    N, C, H, W = _shape_args(x.shape, layout)
    Co, kh, kw = wshape[0], wshape[-2], wshape[-1]
    m = Co // C
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    dw = np.zeros((Co, kh, kw))
    a = np.zeros_like(dw)
    _load().oracle_dw_bwd_filter(_p(x), _p(dy), _p(dw), _p(a), N, C, H, W, m, kh, kw, sh, sw, ph, pw, layout)
    return dw, a


def dense_weights(w, C: int) -> np.ndarray:
    """Eq. 1 generalised to m: [C*m, kh, kw] -> dense block-diagonal [C*m, C, kh, kw]."""
    w = _d(w)
    Co, kh, kw = w.shape
    m = Co // C
    wd = np.zeros((Co, C, kh, kw))
    _load().oracle_expand_weights(_p(w), _p(wd), C, m, kh, kw)
    return wd


def mask(C: int, m: int, kh: int, kw: int) -> np.ndarray:
    a = np.zeros((C * m, C, kh, kw))
    _load().oracle_mask(_p(a), C, m, kh, kw)
    return a


def hadamard(a, b) -> np.ndarray:
    a, b = _d(a), _d(b)
    out = np.zeros_like(a)
    _load().oracle_hadamard(_p(a), _p(b), _p(out), a.size)
    return out


def dense_fwd(x, wd, stride=1, padding=0) -> np.ndarray:
    x, wd = _d(x), _d(wd)
    N, Ci, H, W = x.shape
    Co, _, kh, kw = wd.shape
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    Ho, Wo = out_size(H, kh, sh, ph), out_size(W, kw, sw, pw)
    y = np.zeros((N, Co, Ho, Wo))
    _load().oracle_dense_fwd(_p(x), _p(wd), _p(y), N, Ci, H, W, Co, kh, kw, sh, sw, ph, pw)
    return y


def dense_bwd_data(dy, wd, xshape, stride=1, padding=0) -> np.ndarray:
    dy, wd = _d(dy), _d(wd)
    N, Ci, H, W = xshape
    Co, _, kh, kw = wd.shape
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    dx = np.zeros((N, Ci, H, W))
    _load().oracle_dense_bwd_data(_p(dy), _p(wd), _p(dx), N, Ci, H, W, Co, kh, kw, sh, sw, ph, pw)
    return dx


def dense_bwd_filter(x, dy, wdshape, stride=1, padding=0) -> np.ndarray:
    x, dy = _d(x), _d(dy)
    N, Ci, H, W = x.shape
    Co, _, kh, kw = wdshape
    (kh, kw), (sh, sw), (ph, pw) = _hw((kh, kw), stride, padding)
    g = np.zeros((Co, Ci, kh, kw))
    _load().oracle_dense_bwd_filter(_p(x), _p(dy), _p(g), N, Ci, H, W, Co, kh, kw, sh, sw, ph, pw)
    return g


def round_to(a, dtype: str) -> np.ndarray:
    """Single RNE rounding of double results to the storage dtype ('f32' or 'bf16')."""
    a = _d(a)
    out = np.zeros_like(a)
    _load().oracle_round(_p(a), _p(out), a.size, {"f32": F32, "bf16": BF16}[dtype])
    return out

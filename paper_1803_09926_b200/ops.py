"""Python binding of include/dwconv.h over torch tensors (argument marshalling only).

Names mirror the C ABI (``dwconv_fwd``, ``dwconv_bwd_data``, ``dwconv_bwd_filter``):
they take a descriptor plus device tensors and enqueue on the current torch
stream.  ``fwd`` / ``bwd_data`` / ``bwd_filter`` additionally allocate the output.
Every step of the computation runs in libdwconv.so; torch provides device
memory and the stream.

Layout: tensors are logical ``[N, C, H, W]``; NCHW means ``x.is_contiguous()``,
NHWC means ``x.is_contiguous(memory_format=torch.channels_last)`` (the C ABI's
[N][H][W][C]).  When both hold (C == 1 or H == W == 1) NCHW is used unless
``layout`` says otherwise.
"""
from __future__ import annotations

import ctypes
import threading
from typing import Dict, List, Optional, Sequence, Tuple, Union

import torch

from . import _lib
from ._lib import BF16, F32, NCHW, NHWC, Desc, PlanInfo

IntPair = Union[int, Sequence[int]]


def _pair(v: IntPair) -> Tuple[int, int]:
    if isinstance(v, int):
        return v, v
    a, b = v
    return int(a), int(b)


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return F32
    if t == torch.bfloat16:
        return BF16
    raise TypeError(f"dwconv supports float32 and bfloat16 storage, got {t}")


def infer_layout(x: torch.Tensor, layout: Optional[int] = None) -> int:
    if layout is not None:
        ok = x.is_contiguous() if layout == NCHW else x.is_contiguous(memory_format=torch.channels_last)
        if not ok:
            raise ValueError("tensor memory format does not match the requested layout")
        return layout
    if x.is_contiguous():
        return NCHW
    if x.is_contiguous(memory_format=torch.channels_last):
        return NHWC
    raise ValueError("activations must be contiguous NCHW or channels_last (NHWC)")


def make_desc(n: int, c: int, h: int, w: int, multiplier: int, kernel: IntPair, stride: IntPair = 1,
              padding: IntPair = 0, layout: int = NCHW, dtype: int = F32) -> Desc:
    kh, kw = _pair(kernel)
    sh, sw = _pair(stride)
    ph, pw = _pair(padding)
    return Desc(n, c, h, w, multiplier, kh, kw, sh, sw, ph, pw, layout, dtype)


def output_shape(d: Desc) -> Tuple[int, int]:
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().dwconv_output_shape(ctypes.byref(d), ctypes.byref(ho), ctypes.byref(wo)),
               "dwconv_output_shape")
    return int(ho.value), int(wo.value)


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t: Optional[torch.Tensor]) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _check_dev(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise ValueError("dwconv tensors must be CUDA device tensors (there is no CPU path)")
    devs = {t.device for t in ts}
    if len(devs) > 1:
        raise ValueError(f"dwconv tensors must share one device, got {sorted(str(v) for v in devs)}")


_STORAGE = {F32: torch.float32, BF16: torch.bfloat16}


def _check_tensors(d: Desc, **ts: torch.Tensor) -> None:
    """Match every tensor against the descriptor before its raw pointer reaches the C library (which sees
    no shapes or dtypes): storage dtype, logical [N, C, H, W] / [N, C*m, Ho, Wo] shape, memory format and
    weight size.  A mismatch raises ValueError naming both shapes (SPEC "shape mismatch" is an error)."""
    _check_dev(*ts.values())
    ho, wo = output_shape(d)
    co = d.c * d.multiplier
    want = {"x": (d.n, d.c, d.h, d.w), "dx": (d.n, d.c, d.h, d.w), "y": (d.n, co, ho, wo), "dy": (d.n, co, ho, wo)}
    sdt = _STORAGE[d.dtype]
    for name, t in ts.items():
        if name == "dw":
            if t.dtype != torch.float32:
                raise TypeError("dw is always float32")
            if t.numel() != co * d.kh * d.kw or not t.is_contiguous():
                raise ValueError(f"dw must be a contiguous float32 tensor of {co * d.kh * d.kw} elements "
                                 f"([C*m, kh, kw] = [{co}, {d.kh}, {d.kw}]), got shape {tuple(t.shape)}")
            continue
        if t.dtype != sdt:
            raise TypeError(f"{name} has dtype {t.dtype} but the descriptor's storage dtype is {sdt}")
        if name == "w":
            if t.numel() != co * d.kh * d.kw or not t.is_contiguous():
                raise ValueError(f"w must be a contiguous tensor of {co * d.kh * d.kw} elements "
                                 f"([C*m, kh, kw] = [{co}, {d.kh}, {d.kw}]), got shape {tuple(t.shape)}")
            continue
        if tuple(t.shape) != want[name]:
            raise ValueError(f"{name} has shape {tuple(t.shape)} but the descriptor needs {want[name]}")
        ok = t.is_contiguous() if d.layout == NCHW else t.is_contiguous(memory_format=torch.channels_last)
        if not ok:
            raise ValueError(f"{name} is not contiguous in the descriptor's layout "
                             f"({'NCHW' if d.layout == NCHW else 'NHWC / channels_last'})")


# ----------------------------------------------------------------- raw C mirrors
def dwconv_fwd(d: Desc, x: torch.Tensor, w: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    _check_tensors(d, x=x, w=w, y=y)
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().dwconv_fwd(ctypes.byref(d), _ptr(x), _ptr(w), _ptr(y), _stream(stream)),
                   "dwconv_fwd")


def dwconv_bwd_data(d: Desc, dy: torch.Tensor, w: torch.Tensor, dx: torch.Tensor, stream=None) -> None:
    _check_tensors(d, dy=dy, w=w, dx=dx)
    with torch.cuda.device(dy.device):
        _lib.check(_lib.load().dwconv_bwd_data(ctypes.byref(d), _ptr(dy), _ptr(w), _ptr(dx), _stream(stream)),
                   "dwconv_bwd_data")


def dwconv_bwd_filter_workspace_bytes(d: Desc) -> int:
    return int(_lib.load().dwconv_bwd_filter_workspace_bytes(ctypes.byref(d)))


def dwconv_bwd_filter(d: Desc, x: torch.Tensor, dy: torch.Tensor, dw: torch.Tensor,
                      workspace: Optional[torch.Tensor], stream=None) -> None:
    _check_tensors(d, x=x, dy=dy, dw=dw)
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().dwconv_bwd_filter(ctypes.byref(d), _ptr(x), _ptr(dy), _ptr(dw), _ptr(workspace),
                                                 nbytes, _stream(stream)), "dwconv_bwd_filter")


def dwconv_bwd_workspace_bytes(d: Desc) -> int:
    return int(_lib.load().dwconv_bwd_workspace_bytes(ctypes.byref(d)))


def dwconv_bwd(d: Desc, x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, dx: torch.Tensor, dw: torch.Tensor,
               workspace: Optional[torch.Tensor], stream=None) -> None:
    """Fused backward: dx and dw from one pass over x and dy where the library has a fused kernel."""
    _check_tensors(d, x=x, dy=dy, w=w, dx=dx, dw=dw)
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().dwconv_bwd(ctypes.byref(d), _ptr(x), _ptr(dy), _ptr(w), _ptr(dx), _ptr(dw),
                                          _ptr(workspace), nbytes, _stream(stream)), "dwconv_bwd")


def dwconv_workspace_init(workspace: torch.Tensor, stream=None) -> None:
    _lib.check(_lib.load().dwconv_workspace_init(_ptr(workspace), workspace.numel() * workspace.element_size(),
                                                 _stream(stream)), "dwconv_workspace_init")


def dwconv_plan(d: Desc, pass_: int) -> Dict[str, int]:
    info = PlanInfo()
    _lib.check(_lib.load().dwconv_plan(ctypes.byref(d), pass_, ctypes.byref(info)), "dwconv_plan")
    out = {f: getattr(info, f) for f, _ in PlanInfo._fields_}
    out["variant_name"] = _lib.VARIANTS.get(info.variant, "?")
    return out


def dwconv_plan_candidates(d: Desc, pass_: int, max_candidates: int = _lib.MAX_CANDIDATES) -> List[Dict[str, int]]:
    """Distinct NCHW launch shapes for (d, pass_), the planner's default first (include/dwconv.h)."""
    infos = (PlanInfo * max(1, max_candidates))()
    count = ctypes.c_int32(0)
    _lib.check(_lib.load().dwconv_plan_candidates(ctypes.byref(d), pass_, max_candidates, infos,
                                                  ctypes.byref(count)), "dwconv_plan_candidates")
    out = []
    for i in range(count.value):
        e = {f: getattr(infos[i], f) for f, _ in PlanInfo._fields_}
        e["variant_name"] = _lib.VARIANTS.get(infos[i].variant, "?")
        out.append(e)
    return out


def dwconv_plan_select(d: Desc, pass_: int, index: int) -> None:
    """Install candidate `index` of dwconv_plan_candidates for (d, pass_); -1 restores the default."""
    _lib.check(_lib.load().dwconv_plan_select(ctypes.byref(d), pass_, index), "dwconv_plan_select")


class Plan:
    """An immutable launch plan (``dwconv_plan_create``): descriptor + pass + candidate resolved once.

    ``candidate=-1`` is the planner's own pick; ``k >= 0`` is entry k of ``dwconv_plan_candidates``.  Calls
    through a plan never read process-wide state (``dwconv_plan_select`` does not affect them), so plans
    are safe to share between threads and to capture in CUDA graphs.
    """

    def __init__(self, d: Desc, pass_: int, candidate: int = -1):
        self.desc, self.pass_, self.candidate = d, pass_, candidate
        h = ctypes.c_void_p()
        self._lib = _lib.load()
        _lib.check(self._lib.dwconv_plan_create(ctypes.byref(d), pass_, candidate, ctypes.byref(h)),
                   "dwconv_plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.dwconv_plan_destroy(h)
            self._h = None

    @property
    def workspace_bytes(self) -> int:
        return int(self._lib.dwconv_plan_workspace_bytes(self._h))

    def describe(self) -> Dict[str, int]:
        info = PlanInfo()
        _lib.check(self._lib.dwconv_plan_describe(self._h, ctypes.byref(info)), "dwconv_plan_describe")
        out = {f: getattr(info, f) for f, _ in PlanInfo._fields_}
        out["variant_name"] = _lib.VARIANTS.get(info.variant, "?")
        return out

    def fwd(self, x: torch.Tensor, w: torch.Tensor, y: torch.Tensor, stream=None) -> None:
        _check_tensors(self.desc, x=x, w=w, y=y)
        with torch.cuda.device(x.device):
            _lib.check(self._lib.dwconv_fwd_plan(self._h, _ptr(x), _ptr(w), _ptr(y), _stream(stream)),
                       "dwconv_fwd_plan")

    def bwd_data(self, dy: torch.Tensor, w: torch.Tensor, dx: torch.Tensor, stream=None) -> None:
        _check_tensors(self.desc, dy=dy, w=w, dx=dx)
        with torch.cuda.device(dy.device):
            _lib.check(self._lib.dwconv_bwd_data_plan(self._h, _ptr(dy), _ptr(w), _ptr(dx), _stream(stream)),
                       "dwconv_bwd_data_plan")

    def bwd_filter(self, x: torch.Tensor, dy: torch.Tensor, dw: torch.Tensor, workspace: Optional[torch.Tensor],
                   stream=None) -> None:
        _check_tensors(self.desc, x=x, dy=dy, dw=dw)
        nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        with torch.cuda.device(x.device):
            _lib.check(self._lib.dwconv_bwd_filter_plan(self._h, _ptr(x), _ptr(dy), _ptr(dw), _ptr(workspace),
                                                        nbytes, _stream(stream)), "dwconv_bwd_filter_plan")

    def bwd(self, x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, dx: torch.Tensor, dw: torch.Tensor,
            workspace: Optional[torch.Tensor], stream=None) -> None:
        _check_tensors(self.desc, x=x, dy=dy, w=w, dx=dx, dw=dw)
        nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        with torch.cuda.device(x.device):
            _lib.check(self._lib.dwconv_bwd_plan(self._h, _ptr(x), _ptr(dy), _ptr(w), _ptr(dx), _ptr(dw),
                                                 _ptr(workspace), nbytes, _stream(stream)), "dwconv_bwd_plan")


def dwconv_set_variant_override(v: int) -> None:
    _lib.check(_lib.load().dwconv_set_variant_override(v), "dwconv_set_variant_override")


# ----------------------------------------------------------------- workspaces
class _Workspaces:
    """Zero-initialised bwd_filter workspaces, one per (device, stream).

    The kernel leaves its workspace zeroed, so a buffer is reused by every later
    call on the same stream; it only grows.
    """

    def __init__(self):
        self._mu = threading.Lock()
        self._bufs: Dict[Tuple[int, int], torch.Tensor] = {}

    def get(self, nbytes: int, device: torch.device, stream=None) -> Optional[torch.Tensor]:
        if nbytes == 0:
            return None
        s = stream if stream is not None else torch.cuda.current_stream(device)
        key = (device.index if device.index is not None else torch.cuda.current_device(), s.cuda_stream)
        with self._mu:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.zeros(max(nbytes, 4096), dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


WORKSPACES = _Workspaces()


# ----------------------------------------------------------------- convenience API
def desc_for(x: torch.Tensor, w_shape: Sequence[int], stride: IntPair = 1, padding: IntPair = 0,
             layout: Optional[int] = None) -> Desc:
    lay = infer_layout(x, layout)
    n, c, h, wd = x.shape
    co = int(w_shape[0])
    kh, kw = int(w_shape[-2]), int(w_shape[-1])
    if co % c:
        raise ValueError("weight channels must be a multiple of input channels")
    return make_desc(n, c, h, wd, co // c, (kh, kw), stride, padding, lay, _dtype_code(x.dtype))


def _alloc(shape, like: torch.Tensor, layout: int) -> torch.Tensor:
    mf = torch.channels_last if layout == NHWC else torch.contiguous_format
    return torch.empty(shape, dtype=like.dtype, device=like.device, memory_format=mf)


def fwd(x: torch.Tensor, w: torch.Tensor, stride: IntPair = 1, padding: IntPair = 0,
        layout: Optional[int] = None) -> torch.Tensor:
    """y = depthwise_conv(x, w); w is [C*m, kh, kw] or [C*m, 1, kh, kw]."""
    d = desc_for(x, w.shape, stride, padding, layout)
    ho, wo = output_shape(d)
    y = _alloc((d.n, d.c * d.multiplier, ho, wo), x, d.layout)
    dwconv_fwd(d, x, w.contiguous(), y)
    return y


def bwd_data(dy: torch.Tensor, w: torch.Tensor, x_shape: Sequence[int], stride: IntPair = 1,
             padding: IntPair = 0, layout: Optional[int] = None) -> torch.Tensor:
    lay = infer_layout(dy, layout)
    n, c, h, wd = (int(v) for v in x_shape)
    d = make_desc(n, c, h, wd, int(w.shape[0]) // c, (int(w.shape[-2]), int(w.shape[-1])), stride, padding,
                  lay, _dtype_code(dy.dtype))
    dx = _alloc((n, c, h, wd), dy, lay)
    dwconv_bwd_data(d, dy, w.contiguous(), dx)
    return dx


def bwd_filter(x: torch.Tensor, dy: torch.Tensor, w_shape: Sequence[int], stride: IntPair = 1,
               padding: IntPair = 0, layout: Optional[int] = None) -> torch.Tensor:
    """dw (float32, [C*m, kh, kw]) = sum over batch and space of x (*) dy."""
    d = desc_for(x, w_shape, stride, padding, layout)
    dw = torch.empty((d.c * d.multiplier, d.kh, d.kw), dtype=torch.float32, device=x.device)
    ws = WORKSPACES.get(dwconv_bwd_filter_workspace_bytes(d), x.device)
    dwconv_bwd_filter(d, x, dy, dw, ws)
    return dw


def bwd(x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, stride: IntPair = 1, padding: IntPair = 0,
        layout: Optional[int] = None):
    """(dx, dw) of one layer through the fused backward entry point (dwconv_bwd)."""
    d = desc_for(x, w.shape, stride, padding, layout)
    dx = _alloc((d.n, d.c, d.h, d.w), x, d.layout)
    dw = torch.empty((d.c * d.multiplier, d.kh, d.kw), dtype=torch.float32, device=x.device)
    ws = WORKSPACES.get(dwconv_bwd_workspace_bytes(d), x.device)
    dwconv_bwd(d, x, dy, w.contiguous(), dx, dw, ws)
    return dx, dw


class DepthwiseConv2dFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, stride, padding):
        w3 = w.reshape(w.shape[0], w.shape[-2], w.shape[-1])
        ctx.save_for_backward(x, w3)
        ctx.stride, ctx.padding, ctx.wshape = stride, padding, w.shape
        return fwd(x, w3, stride, padding)

    @staticmethod
    def backward(ctx, dy):
        x, w3 = ctx.saved_tensors
        lay = infer_layout(x)
        mf = torch.channels_last if lay == NHWC else torch.contiguous_format
        dy = dy.contiguous(memory_format=mf)
        dx = dw = None
        if ctx.needs_input_grad[0] and ctx.needs_input_grad[1]:  # one fused pass over x and dy
            dx, dw = bwd(x, dy, w3, ctx.stride, ctx.padding, lay)
            return dx, dw.to(w3.dtype).reshape(ctx.wshape), None, None
        if ctx.needs_input_grad[0]:
            dx = bwd_data(dy, w3, x.shape, ctx.stride, ctx.padding, lay)
        if ctx.needs_input_grad[1]:
            dw = bwd_filter(x, dy, w3.shape, ctx.stride, ctx.padding, lay).to(w3.dtype).reshape(ctx.wshape)
        return dx, dw, None, None


class DepthwiseConv2d(torch.nn.Module):
    """Depthwise conv layer (groups = in_channels, no bias) on the dwconv kernels."""

    def __init__(self, channels: int, kernel_size: int = 3, stride: int = 1, padding: Optional[int] = None,
                 multiplier: int = 1, dtype=torch.float32, device=None):
        super().__init__()
        self.stride = stride
        self.padding = (kernel_size - 1) // 2 if padding is None else padding
        self.weight = torch.nn.Parameter(
            torch.empty(channels * multiplier, 1, kernel_size, kernel_size, dtype=dtype, device=device))
        torch.nn.init.kaiming_uniform_(self.weight, a=5 ** 0.5)

    def forward(self, x):
        return DepthwiseConv2dFn.apply(x, self.weight, self.stride, self.padding)

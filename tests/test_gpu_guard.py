"""Guard bands around every output (a stand-in for compute-sanitizer memcheck, which is closed on
this pool): every candidate plan of every pass writes y / dx / dw into the middle of a larger
allocation whose head and tail hold a sentinel pattern; a single stray store past either end of
the tensor (bulk shared->global stores of the lane kernels, vector stores of partial tiles, the
slice-partial workspace) changes a sentinel.  The interior is also checked, bitwise against the
oracle on small-integer data (exact in any summation order), so a candidate that skips work or
writes the wrong element fails too.  Shapes: the round-3 kernel families at small batch --
bf16 112x112 stride 1 / 2 (interleaved strips, streaming stride-2 input gradient, producer-warp
and streaming filter gradients), 56x56, 14x14 and 7x7 lane-per-plane planes, both dtypes.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1803_09926_b200 import ops
from paper_1803_09926_b200._lib import BF16, F32, NCHW

pytestmark = pytest.mark.gpu

PAD = 4096  # elements of guard band on each side (16-B multiple in both dtypes)
SENT = -1536.0  # exact in bf16 and fp32

SHAPES = [  # N, C, H, m, K, s, p
    (2, 32, 112, 1, 3, 1, 1),
    (2, 32, 112, 1, 3, 2, 1),
    (2, 64, 56, 1, 3, 1, 1),
    (4, 64, 14, 1, 3, 1, 1),
    (4, 64, 7, 1, 3, 1, 1),
]


def _guarded(n_elems, dtype, device="cuda"):
    buf = torch.full((PAD + n_elems + PAD,), SENT, dtype=dtype, device=device)
    return buf, buf[PAD:PAD + n_elems]


def _check_guards(buf, n_elems, tag):
    head = buf[:PAD].float().cpu().numpy()
    tail = buf[PAD + n_elems:].float().cpu().numpy()
    assert np.all(head == SENT) and np.all(tail == SENT), f"{tag}: store outside the tensor"


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"N{s[0]}C{s[1]}H{s[2]}s{s[5]}")
def test_guard_bands_every_candidate(shape, dtype):
    N, C, H, m, K, s, p = shape
    W = H
    Ho = (H + 2 * p - K) // s + 1
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    xs = synth.integers(11, (N, C, H, W), 3)
    ws = synth.integers(12, (C * m, K, K), 3)
    dys = synth.integers(13, (N, C * m, Ho, Ho), 3)
    x = torch.from_numpy(xs.astype(np.float32)).to(tdt).cuda()
    w = torch.from_numpy(ws.astype(np.float32)).to(tdt).cuda()
    dy = torch.from_numpy(dys.astype(np.float32)).to(tdt).cuda()
    f64 = np.float64
    ref_y = oracle.fwd(xs.astype(f64), ws.astype(f64), s, p)[0]
    ref_dx = oracle.bwd_data(dys.astype(f64), ws.astype(f64), xs.shape, s, p)[0]
    ref_dw = oracle.bwd_filter(xs.astype(f64), dys.astype(f64), ws.shape, s, p)[0]
    d = ops.make_desc(N, C, H, W, m, K, s, p, NCHW, F32 if dtype == "f32" else BF16)
    ny, nx, nw = dy.numel(), x.numel(), C * m * K * K
    for name, pas in (("fwd", 0), ("bwd_data", 1), ("bwd_filter", 2)):
        cands = ops.dwconv_plan_candidates(d, pas) or [None]
        for i, c in enumerate(cands):
            pl = ops.Plan(d, pas, i if c is not None else -1)
            tag = f"{name} candidate {i} ({c['kernel_family'] if c else '-'})"
            if pas == 0:
                buf, y = _guarded(ny, tdt)
                pl.fwd(x, w, y.view(dy.shape))
                torch.cuda.synchronize()
                _check_guards(buf, ny, tag)
                assert np.array_equal(y.view(dy.shape).float().cpu().numpy().astype(f64), ref_y), tag
            elif pas == 1:
                buf, dx = _guarded(nx, tdt)
                pl.bwd_data(dy, w, dx.view(x.shape))
                torch.cuda.synchronize()
                _check_guards(buf, nx, tag)
                assert np.array_equal(dx.view(x.shape).float().cpu().numpy().astype(f64), ref_dx), tag
            else:
                buf, dwt = _guarded(nw, torch.float32)
                wsb = max(16, pl.workspace_bytes)
                wbuf = torch.zeros(PAD * 2 + wsb, dtype=torch.uint8, device="cuda")
                wbuf[:PAD].fill_(0x5A)
                wbuf[PAD + wsb:].fill_(0x5A)
                pl.bwd_filter(x, dy, dwt.view(C * m, K, K), wbuf[PAD:PAD + wsb])
                torch.cuda.synchronize()
                _check_guards(buf, nw, tag)
                wb = wbuf.cpu().numpy()
                assert np.all(wb[:PAD] == 0x5A) and np.all(wb[PAD + wsb:] == 0x5A), f"{tag}: workspace overrun"
                assert np.all(wb[PAD:PAD + wsb] == 0), f"{tag}: workspace not handed back zeroed"
                assert np.array_equal(dwt.view(C * m, K, K).cpu().numpy().astype(f64), ref_dw), tag


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("dtype,batch", [("f32", 64), ("bf16", 128)])
def test_candidate_lists_capped(dtype, batch, layout):
    """Every MobileNet layer's candidate list (count query with max_candidates = 0 included) stays within
    DWCONV_MAX_CANDIDATES, and every listed index builds a plan handle (include/dwconv.h)."""
    from paper_1803_09926_b200 import _lib
    import ctypes
    lib = _lib.load()
    for L in synth.mobilenet_v1_dw(batch):
        d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout, F32 if dtype == "f32" else BF16)
        for pas in (0, 1, 2):
            count = ctypes.c_int(-1)
            rc = lib.dwconv_plan_candidates(ctypes.byref(d), pas, 0, None, ctypes.byref(count))
            assert rc == 0 and 0 <= count.value <= _lib.MAX_CANDIDATES, (L.name, pas, count.value)
            cands = ops.dwconv_plan_candidates(d, pas)
            assert len(cands) == count.value
            for i in range(len(cands)):
                ops.Plan(d, pas, i)

"""GPU parity at BASELINE.json's full sizes, in the launch configurations bench.py
can time: every candidate plan the library offers (``dwconv_plan_candidates``,
which ``tune.py`` chooses among before the bench's timed region), for every
MobileNet-v1 depthwise layer at batch 64 (configs[1], fp32 NCHW) and the
large layers at batch 128 in bf16 (configs[2]).

Inputs are small integers ({-4..4} at b64 fp32, {-2..2}
at b128 bf16), so every sum is exact in any order and the CUDA result must
equal the oracle BITWISE (rule R1).  The oracle computes sampled outputs one
by one: whole (n, c) output planes for fwd / bwd_data (each depends on one
input plane), and whole channels of dw for bwd_filter (each depends on that
channel's planes over the full batch).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1803_09926_b200 import ops
from paper_1803_09926_b200._lib import F32, BF16, NCHW, NHWC

pytestmark = pytest.mark.gpu

NSAMP = 6


def _dev(a, dtype, layout=NCHW):
    t = torch.from_numpy(a)
    t = (t.to(torch.bfloat16) if dtype == "bf16" else t).cuda()
    return t.contiguous(memory_format=torch.channels_last) if (layout == NHWC and t.dim() == 4) else t


def _check_layer(L, dtype, amax, seed, layout=NCHW):
    rng = np.random.default_rng(seed)
    x = synth.integers(seed * 10 + 1, (L.n, L.c, L.h, L.w), amax)
    w = synth.integers(seed * 10 + 2, (L.c * L.m, L.k, L.k), amax)
    dy = synth.integers(seed * 10 + 3, (L.n, L.c * L.m, L.ho, L.wo), amax)
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout, F32 if dtype == "f32" else BF16)
    xd, wd, dyd = _dev(x, dtype, layout), _dev(w, dtype), _dev(dy, dtype, layout)
    y = torch.empty_like(dyd)
    dx = torch.empty_like(xd)
    dwt = torch.empty(w.shape, dtype=torch.float32, device="cuda")
    planes = [(int(rng.integers(L.n)), int(rng.integers(L.c))) for _ in range(NSAMP)]
    chans = sorted({int(c) for c in rng.integers(L.c, size=NSAMP)})
    s, p = L.s, L.p
    ref = {"fwd": {}, "bwd_data": {}, "bwd_filter": {}}
    for n, c in planes:
        ref["fwd"][(n, c)] = oracle.fwd(x[n:n + 1, c:c + 1].astype(np.float64),
                                        w[c:c + 1].astype(np.float64), s, p)[0][0, 0]
        ref["bwd_data"][(n, c)] = oracle.bwd_data(dy[n:n + 1, c:c + 1].astype(np.float64),
                                                  w[c:c + 1].astype(np.float64), (1, 1, L.h, L.w), s, p)[0][0, 0]
    for c in chans:
        ref["bwd_filter"][c] = oracle.bwd_filter(x[:, c:c + 1].astype(np.float64), dy[:, c:c + 1].astype(np.float64),
                                                 (1, L.k, L.k), s, p)[0][0]
    for name, pas in (("fwd", 0), ("bwd_data", 1), ("bwd_filter", 2)):
        cands = ops.dwconv_plan_candidates(d, pas)
        if not cands:  # shapes only the generic kernels cover: check the default path once
            assert layout == NHWC or L.c < 4 or L.n == 0, f"{L.name} {name}: no candidates"
            cands = [None]
        ws = None
        if pas == 2:
            ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d),
                                 max((c["workspace_bytes"] for c in cands if c), default=0)),
                             dtype=torch.uint8, device="cuda")
        try:
            for i, cand in enumerate(cands):
                if cand is not None:
                    ops.dwconv_plan_select(d, pas, i)
                tag = f"{L.name} {dtype} {name} candidate {i} {cand}"
                if pas == 0:
                    y.fill_(float("nan"))
                    ops.dwconv_fwd(d, xd, wd, y)
                    for (n, c), r in ref["fwd"].items():
                        got = y[n, c].float().cpu().numpy()
                        assert np.array_equal(got, r.astype(np.float32)), tag
                elif pas == 1:
                    dx.fill_(float("nan"))
                    ops.dwconv_bwd_data(d, dyd, wd, dx)
                    for (n, c), r in ref["bwd_data"].items():
                        got = dx[n, c].float().cpu().numpy()
                        assert np.array_equal(got, r.astype(np.float32)), tag
                else:
                    dwt.fill_(float("nan"))
                    ops.dwconv_bwd_filter(d, xd, dyd, dwt, ws)
                    got = dwt.cpu().numpy()
                    for c, r in ref["bwd_filter"].items():
                        assert np.array_equal(got[c], r.astype(np.float32)), tag
        finally:
            ops.dwconv_plan_select(d, pas, -1)
    # fused backward (dwconv_bwd: dx and dw from one pass) where the library has it
    if layout == NCHW and ops.dwconv_plan(d, 3)["variant_name"] != "none":
        cands = ops.dwconv_plan_candidates(d, 3)
        ws = torch.zeros(max(16, max(c["workspace_bytes"] for c in cands)), dtype=torch.uint8, device="cuda")
        try:
            for i, cand in enumerate(cands):
                ops.dwconv_plan_select(d, 3, i)
                tag = f"{L.name} {dtype} bwd (fused) candidate {i} {cand}"
                dx.fill_(float("nan"))
                dwt.fill_(float("nan"))
                ops.dwconv_bwd(d, xd, dyd, wd, dx, dwt, ws)
                for (n, c), r in ref["bwd_data"].items():
                    assert np.array_equal(dx[n, c].float().cpu().numpy(), r.astype(np.float32)), tag
                got = dwt.cpu().numpy()
                for c, r in ref["bwd_filter"].items():
                    assert np.array_equal(got[c], r.astype(np.float32)), tag
        finally:
            ops.dwconv_plan_select(d, 3, -1)
    torch.cuda.synchronize()


@pytest.mark.parametrize("layer", [L.name for L in synth.mobilenet_v1_dw(64)])
def test_candidates_fullsize_b64_fp32(layer):
    L = [l for l in synth.mobilenet_v1_dw(64) if l.name == layer][0]
    _check_layer(L, "f32", 4, seed=7)


@pytest.mark.parametrize("layer", ["dw2", "dw4", "dw8", "dw14", "dw24", "dw26"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_candidates_fullsize_nhwc(layer, dtype):
    """NHWC: every TMA / register-tile candidate at the bench's sizes (b64 fp32, b128 bf16)."""
    L = [l for l in synth.mobilenet_v1_dw(64 if dtype == "f32" else 128) if l.name == layer][0]
    _check_layer(L, dtype, 4 if dtype == "f32" else 2, seed=9, layout=NHWC)


@pytest.mark.parametrize("layer", ["dw2", "dw4", "dw14", "dw26"])
def test_candidates_fullsize_b128_bf16(layer):
    L = [l for l in synth.mobilenet_v1_dw(128) if l.name == layer][0]
    _check_layer(L, "bf16", 2, seed=8)


def test_tune_layer_selects_a_candidate():
    from paper_1803_09926_b200 import tune
    L = [l for l in synth.mobilenet_v1_dw(16) if l.name == "dw14"][0]
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NCHW, F32)
    x = torch.randn(L.n, L.c, L.h, L.w, device="cuda")
    dy = torch.randn(L.n, L.c, L.ho, L.wo, device="cuda")
    w = torch.randn(L.c, L.k, L.k, device="cuda")
    res = tune.tune_layer(d, x, dy, w)
    try:
        assert set(res) == {"fwd", "bwd_data", "bwd_filter"}
        for name, r in res.items():
            assert 0 <= r["index"] < r["candidates"] and r["us"] <= r["default_us"]
            info = ops.dwconv_plan(d, tune.PASSES[name])
            assert info["grid"] == r["grid"] and info["block"] == r["block"]
    finally:
        for p in range(3):
            ops.dwconv_plan_select(d, p, -1)


# Edge shapes for the small-plane / band / TMA candidates at small batch: one
# channel group, channel counts that do not fill a CTA, single-image slices,
# stride 2 on 14 / 28 planes, and the band kernel's one- and two-plane warps.
EDGE = [
    # (N, C, H, s)
    (1, 4, 14, 1), (3, 12, 14, 1), (2, 8, 28, 1), (5, 4, 7, 1), (2, 20, 7, 1),
    (3, 8, 14, 2), (2, 12, 28, 2),
    (2, 6, 56, 1), (1, 3, 112, 1), (2, 4, 112, 2), (3, 5, 56, 2), (2, 2, 28, 1),
]


@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", EDGE)
def test_candidates_edge_shapes(shape, dtype, layout):
    n, c, h, s = shape
    L = synth.Layer(name=f"edge{n}x{c}x{h}s{s}", n=n, c=c, h=h, w=h, k=3, s=s, p=1, m=1)
    _check_layer(L, dtype, 3 if dtype == "f32" else 2, seed=11, layout=layout)

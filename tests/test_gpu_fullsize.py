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


def _inputs(L, dtype, kind, amax, seed):
    shapes = ((L.n, L.c, L.h, L.w), (L.c * L.m, L.k, L.k), (L.n, L.c * L.m, L.ho, L.wo))
    if kind == "int":
        return [synth.integers(seed * 10 + i + 1, shp, amax) for i, shp in enumerate(shapes)]
    return [synth.uniform(seed * 10 + i + 1, shp, dtype) for i, shp in enumerate(shapes)]


def _cmp(got, ref, absum, dtype, kind, tag):
    """R1 (integers: bitwise) or R2 / R3 (uniform: |gpu - ref| <= 1e-5 sum|t| (+ 1e-2 |ref| for bf16 storage),
    exact zero where every term is zero)."""
    if kind == "int":
        assert np.array_equal(got, ref.astype(np.float32)), tag
        return
    tol = 1e-5 * absum + (1e-2 * np.abs(ref) if dtype == "bf16" else 0.0)
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= tol), f"{tag}: {int((err > tol).sum())} outside, worst {np.max(err - tol):.3e}"
    assert np.all(got[absum == 0] == 0), tag


def _check_layer(L, dtype, amax, seed, layout=NCHW, kind="int"):
    """Every candidate plan of every pass of layer L (and the fused backward where the library has it)
    against oracle outputs computed one by one on sampled (n, c) planes / dw channels (any m, K, s)."""
    rng = np.random.default_rng(seed)
    x, w, dy = _inputs(L, dtype, kind, amax, seed)
    m = L.m
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout, F32 if dtype == "f32" else BF16)
    xd, wd, dyd = _dev(x, dtype, layout), _dev(w, dtype), _dev(dy, dtype, layout)
    y = torch.empty_like(dyd)
    dx = torch.empty_like(xd)
    dwt = torch.empty(w.shape, dtype=torch.float32, device="cuda")
    planes = [(int(rng.integers(L.n)), int(rng.integers(L.c))) for _ in range(NSAMP)]
    chans = sorted({int(c) for c in rng.integers(L.c, size=NSAMP)})
    s, p = L.s, L.p
    ref = {"fwd": {}, "bwd_data": {}, "bwd_filter": {}}
    f64 = np.float64
    for n, c in planes:
        wc = w[c * m:(c + 1) * m].astype(f64)
        yv, ya = oracle.fwd(x[n:n + 1, c:c + 1].astype(f64), wc, s, p)
        ref["fwd"][(n, c)] = (yv[0], ya[0])
        dv, da = oracle.bwd_data(dy[n:n + 1, c * m:(c + 1) * m].astype(f64), wc, (1, 1, L.h, L.w), s, p)
        ref["bwd_data"][(n, c)] = (dv[0, 0], da[0, 0])
    for c in chans:
        ref["bwd_filter"][c] = oracle.bwd_filter(x[:, c:c + 1].astype(f64), dy[:, c * m:(c + 1) * m].astype(f64),
                                                 (m, L.k, L.k), s, p)

    def check_y(tag):
        for (n, c), (r, a) in ref["fwd"].items():
            _cmp(y[n, c * m:(c + 1) * m].float().cpu().numpy(), r, a, dtype, kind, tag)

    def check_dx(tag):
        for (n, c), (r, a) in ref["bwd_data"].items():
            _cmp(dx[n, c].float().cpu().numpy(), r, a, dtype, kind, tag)

    def check_dw(tag):
        got = dwt.cpu().numpy()
        for c, (r, a) in ref["bwd_filter"].items():
            _cmp(got[c * m:(c + 1) * m], r, a, "f32", kind, tag)

    for name, pas in (("fwd", 0), ("bwd_data", 1), ("bwd_filter", 2)):
        cands = ops.dwconv_plan_candidates(d, pas)
        if not cands:  # shapes only the generic kernels cover: check the default path once
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
                tag = f"{L.name} {dtype} {kind} {name} candidate {i} {cand}"
                if pas == 0:
                    y.fill_(float("nan"))
                    ops.dwconv_fwd(d, xd, wd, y)
                    check_y(tag)
                elif pas == 1:
                    dx.fill_(float("nan"))
                    ops.dwconv_bwd_data(d, dyd, wd, dx)
                    check_dx(tag)
                else:
                    dwt.fill_(float("nan"))
                    ops.dwconv_bwd_filter(d, xd, dyd, dwt, ws)
                    check_dw(tag)
        finally:
            ops.dwconv_plan_select(d, pas, -1)
    # fused backward (dwconv_bwd: dx and dw from one pass) where the library has it
    if ops.dwconv_plan(d, 3)["variant_name"] != "none":
        cands = ops.dwconv_plan_candidates(d, 3) or [None]
        ws = torch.zeros(max(16, ops.dwconv_bwd_workspace_bytes(d),
                             max((c["workspace_bytes"] for c in cands if c), default=0)),
                         dtype=torch.uint8, device="cuda")
        try:
            for i, cand in enumerate(cands):
                if cand is not None:
                    ops.dwconv_plan_select(d, 3, i)
                tag = f"{L.name} {dtype} {kind} bwd (fused) candidate {i} {cand}"
                dx.fill_(float("nan"))
                dwt.fill_(float("nan"))
                ops.dwconv_bwd(d, xd, dyd, wd, dx, dwt, ws)
                check_dx(tag)
                check_dw(tag)
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


@pytest.mark.parametrize("layer", [L.name for L in synth.mobilenet_v1_dw(64)])
def test_candidates_fullsize_b64_fp32_uniform(layer):
    """Random U[-1,1] data at the bench's size (configs[1]) over every tuned candidate: R2 on the sampled
    outputs, i.e. the rounding of the full 802,816-term dw sums, not only their indexing."""
    L = [l for l in synth.mobilenet_v1_dw(64) if l.name == layer][0]
    _check_layer(L, "f32", 0, seed=17, kind="unif")


@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("layer", [L.name for L in synth.mobilenet_v1_dw(128)])
def test_candidates_fullsize_b128_bf16_uniform(layer, layout):
    """bf16 storage, U[-1,1], batch 128 (the >= 70 % target set): R3 over every candidate, both layouts."""
    L = [l for l in synth.mobilenet_v1_dw(128) if l.name == layer][0]
    _check_layer(L, "bf16", 0, seed=18, layout=layout, kind="unif")


@pytest.mark.parametrize("layer", ["dw2", "dw4", "dw6", "dw10", "dw14", "dw24", "dw26"])
def test_candidates_fullsize_b128_fp32_uniform(layer):
    L = [l for l in synth.mobilenet_v1_dw(128) if l.name == layer][0]
    _check_layer(L, "f32", 0, seed=19, kind="unif")


# configs[3] stress shapes at the bench size (N=64): m = 2/4, K = 5/7 on 56x56x128; stride 2 on 56x56x512
CFG4 = [synth.Layer("m2", 64, 128, 56, 56, k=3, s=1, p=1, m=2), synth.Layer("m4", 64, 128, 56, 56, k=3, s=1, p=1, m=4),
        synth.Layer("k5", 64, 128, 56, 56, k=5, s=1, p=2, m=1), synth.Layer("k7", 64, 128, 56, 56, k=7, s=1, p=3, m=1),
        synth.Layer("s2k3", 64, 512, 56, 56, k=3, s=2, p=1, m=1),
        synth.Layer("s2k5", 64, 512, 56, 56, k=5, s=2, p=2, m=1),
        synth.Layer("s2k7", 64, 512, 56, 56, k=7, s=2, p=3, m=1)]


@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", [L.name for L in CFG4])
def test_cfg4_fullsize(shape, dtype, layout, kind):
    L = [l for l in CFG4 if l.name == shape][0]
    # integer sets of SURVEY c.6: {-1,0,1} keeps bf16 m*K^2 <= 196 <= 256 and every sum < 2^24
    _check_layer(L, dtype, 1, seed=21, layout=layout, kind=kind)


def test_tune_layer_selects_a_candidate():
    from paper_1803_09926_b200 import tune
    L = [l for l in synth.mobilenet_v1_dw(16) if l.name == "dw14"][0]
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NCHW, F32)
    x = torch.randn(L.n, L.c, L.h, L.w, device="cuda")
    dy = torch.randn(L.n, L.c, L.ho, L.wo, device="cuda")
    w = torch.randn(L.c, L.k, L.k, device="cuda")
    before = {p: ops.dwconv_plan(d, p) for p in range(3)}
    res = tune.tune_layer(d, x, dy, w)
    assert set(res) == {"fwd", "bwd_data", "bwd_filter"}
    for name, r in res.items():
        assert 0 <= r["index"] < r["candidates"] and r["us"] <= r["default_us"]
        info = r["plan"].describe()
        assert info["grid"] == r["grid"] and info["block"] == r["block"]
        # tuning installs nothing process-wide: the descriptor API still runs the planner's pick
        assert ops.dwconv_plan(d, tune.PASSES[name]) == before[tune.PASSES[name]]


def test_plan_handles_match_selected_descriptor_calls_and_ignore_selection():
    """dwconv_plan_create(d, pass, k) launches exactly what dwconv_plan_select(d, pass, k) + the descriptor call
    launches (bitwise equal outputs), and a later dwconv_plan_select does not change what a handle runs."""
    L = [l for l in synth.mobilenet_v1_dw(8) if l.name == "dw6"][0]
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NCHW, F32)
    x = torch.randn(L.n, L.c, L.h, L.w, device="cuda")
    dy = torch.randn(L.n, L.c, L.ho, L.wo, device="cuda")
    w = torch.randn(L.c, L.k, L.k, device="cuda")
    for pas in (0, 1, 2):
        cands = ops.dwconv_plan_candidates(d, pas)
        assert len(cands) >= 2
        for k in (0, len(cands) // 2, len(cands) - 1):
            pl = ops.Plan(d, pas, k)
            assert pl.describe()["grid"] == cands[k]["grid"]
            other = (k + 1) % len(cands)
            ws = torch.zeros(max(16, pl.workspace_bytes, cands[other]["workspace_bytes"]), dtype=torch.uint8,
                             device="cuda")
            try:
                ops.dwconv_plan_select(d, pas, k)
                if pas == 0:
                    a, b = torch.empty_like(dy), torch.empty_like(dy)
                    ops.dwconv_fwd(d, x, w, a)
                    ops.dwconv_plan_select(d, pas, other)
                    pl.fwd(x, w, b)
                elif pas == 1:
                    a, b = torch.empty_like(x), torch.empty_like(x)
                    ops.dwconv_bwd_data(d, dy, w, a)
                    ops.dwconv_plan_select(d, pas, other)
                    pl.bwd_data(dy, w, b)
                else:
                    a, b = torch.empty(w.shape, device="cuda"), torch.empty(w.shape, device="cuda")
                    ops.dwconv_bwd_filter(d, x, dy, a, ws)
                    ops.dwconv_plan_select(d, pas, other)
                    pl.bwd_filter(x, dy, b, ws)
                torch.cuda.synchronize()
                assert torch.equal(a, b), (pas, k)
            finally:
                ops.dwconv_plan_select(d, pas, -1)
    # a pass mismatch is an error, not a silent launch
    pl = ops.Plan(d, 0, -1)
    with pytest.raises(RuntimeError):
        ops._lib.check(ops._lib.load().dwconv_bwd_data_plan(pl._h, dy.data_ptr(), w.data_ptr(), x.data_ptr(),
                                                            None), "mismatch")


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

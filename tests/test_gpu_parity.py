"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Contract: bitwise on small-integer inputs;
|gpu - ref| <= 1e-5 * sum|terms| for fp32 random data; bf16 storage adds
1e-2 * |ref|; dw (always fp32) uses the fp32 rule.  Bitwise run-to-run
determinism.  Shapes span several chunks/tiles with ragged tails, band mode,
the generic path, m > 1, K in {3,5,7}, s in {1,2}, both layouts and dtypes.
"""
import numpy as np
import pytest
import torch

from gpu_util import NCHW, NHWC, check_all, make_inputs, run_gpu, run_oracle, to_dev, check_close

pytestmark = pytest.mark.gpu

LAYOUTS = [NCHW, NHWC]
DTYPES = ["f32", "bf16"]

# (N, C, H, W, m, K, s, p)
CFG1 = (2, 8, 16, 16, 1, 3, 1, 1)
SHAPES = [
    CFG1,
    (3, 5, 13, 11, 1, 3, 2, 1),     # ragged, stride 2, odd sizes
    (2, 6, 14, 14, 2, 3, 1, 1),     # m = 2, W = 14 (not 16-B rows)
    (2, 3, 7, 7, 4, 3, 1, 1),       # m = 4, 7x7 planes
    (2, 4, 12, 10, 1, 5, 1, 2),     # K = 5
    (1, 3, 15, 9, 1, 7, 1, 3),      # K = 7
    (2, 3, 17, 12, 1, 5, 2, 2),     # K = 5, s = 2
    (1, 2, 19, 16, 2, 7, 2, 3),     # K = 7, s = 2, m = 2
    (2, 3, 80, 80, 1, 3, 1, 1),     # band mode (plane + outputs > stage budget)
    (2, 2, 96, 72, 1, 3, 2, 1),     # band mode, stride 2
    (3, 40, 7, 7, 1, 3, 1, 1),      # many small planes, ragged plane groups
]
GENERIC_SHAPES = [
    (2, 3, 9, 11, 1, 2, 3, 0),      # even kernel, stride 3
    (1, 2, 6, 8, 3, 3, 1, 0),       # m = 3, no padding
    (2, 3, 8, 9, 1, 3, 2, 2),       # padding larger than (K-1)/2
]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import paper_1803_09926_b200 as dw
    dw.dwconv_set_variant_override(0)
    yield dw
    dw.dwconv_set_variant_override(0)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("shape", SHAPES + GENERIC_SHAPES)
def test_parity_random(shape, layout, dtype):
    check_all(*shape, layout=layout, dtype=dtype, kind="unif")


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("shape", SHAPES + GENERIC_SHAPES)
def test_parity_integers_bitwise(shape, layout, dtype):
    amax = 2 if dtype == "bf16" else 3
    if dtype == "bf16" and shape[5] == 7:
        amax = 1  # keep |y|, |dx| <= 256 so bf16 stores are exact (SURVEY c.6)
    check_all(*shape, layout=layout, dtype=dtype, kind="int", amax=amax)


@pytest.mark.parametrize("shape", [CFG1, SHAPES[1], SHAPES[8]])
def test_generic_override_matches_oracle(shape, _lib):
    _lib.dwconv_set_variant_override(1)
    try:
        check_all(*shape, layout=NCHW, dtype="f32", kind="int")
        check_all(*shape, layout=NCHW, dtype="f32", kind="unif")
    finally:
        _lib.dwconv_set_variant_override(0)


def test_determinism_bitwise(_lib):
    inp = make_inputs(4, 32, 56, 56, 1, 3, 1, 1, seed=3)
    a = run_gpu(inp, 1, 1, NCHW, "f32")
    b = run_gpu(inp, 1, 1, NCHW, "f32")
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_workspace_reuse_and_zeroed(_lib):
    """Two back-to-back bwd_filter calls share one workspace; it is zero afterwards."""
    import paper_1803_09926_b200.ops as ops
    inp = make_inputs(8, 16, 28, 28, 1, 3, 2, 1, kind="int", seed=5)
    x, dy = to_dev(inp["x"], NCHW, "f32"), to_dev(inp["dy"], NCHW, "f32")
    d = ops.desc_for(x, inp["w"].shape, 2, 1)
    nbytes = ops.dwconv_bwd_filter_workspace_bytes(d)
    ws = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(3):
        dwt = torch.empty(inp["w"].shape, dtype=torch.float32, device="cuda")
        ops.dwconv_bwd_filter(d, x, dy, dwt, ws)
        outs.append(dwt.cpu().numpy())
    torch.cuda.synchronize()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    plan = ops.dwconv_plan(d, 2)
    assert plan["variant_name"] == "nchw_chunk"
    assert ws.sum().item() == 0  # tickets and partials are handed back zeroed
    _, _, (ref, _) = run_oracle(inp, 2, 1)
    assert np.array_equal(outs[0].astype(np.float64), ref)


def test_workspace_shared_across_shapes(_lib):
    """One workspace buffer serves calls with different plans (group counts) in a row."""
    import paper_1803_09926_b200.ops as ops
    shapes = [(2, 3, 80, 80, 1, 3, 1, 1), (3, 40, 7, 7, 1, 3, 1, 1), (2, 8, 16, 16, 1, 3, 1, 1),
              (4, 64, 14, 14, 1, 3, 2, 1), (3, 40, 7, 7, 1, 3, 1, 1)]
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    for i, sh in enumerate(shapes):
        N, C, H, W, m, K, s, p = sh
        inp = make_inputs(*sh, kind="int", seed=20 + i)
        x, dy = to_dev(inp["x"], NCHW, "f32"), to_dev(inp["dy"], NCHW, "f32")
        d = ops.desc_for(x, inp["w"].shape, s, p)
        assert ops.dwconv_bwd_filter_workspace_bytes(d) <= ws.numel()
        dwt = torch.empty(inp["w"].shape, dtype=torch.float32, device="cuda")
        ops.dwconv_bwd_filter(d, x, dy, dwt, ws)
        _, _, (ref, _) = run_oracle(inp, s, p)
        assert np.array_equal(dwt.cpu().numpy().astype(np.float64), ref), sh
    assert ws.sum().item() == 0


def test_workspace_too_small_errors(_lib):
    import paper_1803_09926_b200.ops as ops
    x = torch.zeros(2, 8, 16, 16, device="cuda")
    dy = torch.zeros(2, 8, 16, 16, device="cuda")
    d = ops.desc_for(x, (8, 3, 3), 1, 1)
    need = ops.dwconv_bwd_filter_workspace_bytes(d)
    assert need > 0
    dwt = torch.empty(8, 3, 3, device="cuda")
    with pytest.raises(_lib.DwconvError) as e:
        ops.dwconv_bwd_filter(d, x, dy, dwt, torch.zeros(need - 16, dtype=torch.uint8, device="cuda"))
    assert e.value.status == 5


def test_empty_batch(_lib):
    x = torch.zeros(0, 4, 8, 8, device="cuda")
    w = torch.ones(4, 3, 3, device="cuda")
    y = _lib.fwd(x, w, 1, 1)
    assert y.shape == (0, 4, 8, 8)
    dwt = _lib.bwd_filter(x, torch.zeros(0, 4, 8, 8, device="cuda"), w.shape, 1, 1)
    torch.cuda.synchronize()
    assert dwt.shape == (4, 3, 3) and not dwt.any()


@pytest.mark.parametrize("layout", LAYOUTS)
def test_unaligned_base_pointers(layout, _lib):
    """Tensors starting 4 bytes past a 16-B boundary take the cooperative-copy path."""
    N, C, H, W, m, K, s, p = (2, 8, 14, 14, 1, 3, 1, 1)
    inp = make_inputs(N, C, H, W, m, K, s, p, kind="int", seed=7)

    def shifted(a):
        flat = torch.zeros(a.size + 1, dtype=torch.float32, device="cuda")
        t = flat[1:].view(*a.shape)
        t.copy_(torch.from_numpy(a))
        assert t.data_ptr() % 16 == 4
        return t

    x, dy, w = shifted(inp["x"]), shifted(inp["dy"]), to_dev(inp["w"], NCHW, "f32")
    if layout == NHWC:
        pytest.skip("channels_last views of an offset buffer are not contiguous views")
    y = _lib.fwd(x, w, s, p)
    dx = _lib.bwd_data(dy, w, x.shape, s, p)
    dwt = _lib.bwd_filter(x, dy, w.shape, s, p)
    torch.cuda.synchronize()
    (ry, _), (rdx, _), (rdw, _) = run_oracle(inp, s, p)
    assert np.array_equal(y.cpu().numpy(), ry) and np.array_equal(dx.cpu().numpy(), rdx)
    assert np.array_equal(dwt.cpu().numpy(), rdw)


def test_autograd_module_matches_oracle(_lib):
    inp = make_inputs(2, 8, 16, 16, 1, 3, 1, 1, kind="int", seed=9)
    x = to_dev(inp["x"], NCHW, "f32").requires_grad_(True)
    mod = _lib.DepthwiseConv2d(8, 3, 1, device="cuda")
    with torch.no_grad():
        mod.weight.copy_(torch.from_numpy(inp["w"]).reshape(8, 1, 3, 3))
    y = mod(x)
    y.backward(to_dev(inp["dy"], NCHW, "f32"))
    (ry, _), (rdx, _), (rdw, _) = run_oracle(inp, 1, 1)
    assert np.array_equal(y.detach().cpu().numpy(), ry)
    assert np.array_equal(x.grad.cpu().numpy(), rdx)
    assert np.array_equal(mod.weight.grad.reshape(8, 3, 3).cpu().numpy(), rdw)


def test_plan_selects_fast_path_for_mobilenet(_lib):
    import synth
    import paper_1803_09926_b200.ops as ops
    for L in synth.mobilenet_v1_dw(64):
        d = ops.make_desc(L.n, L.c, L.h, L.w, 1, 3, L.s, 1, NCHW, 0)
        for pas in (0, 1, 2):
            info = ops.dwconv_plan(d, pas)
            assert info["variant_name"] == "nchw_chunk", (L, pas, info)
            if pas == 2:
                assert info["max_chain"] <= 160, (L, info)


def test_bad_descriptor_errors(_lib):
    import paper_1803_09926_b200.ops as ops
    x = torch.zeros(1, 2, 4, 4, device="cuda")
    w = torch.zeros(2, 5, 5, device="cuda")
    y = torch.zeros(1, 2, 4, 4, device="cuda")
    d = ops.make_desc(1, 2, 4, 4, 1, 5, 1, 0)
    with pytest.raises(_lib.DwconvError) as e:
        ops.dwconv_fwd(d, x, w, y)
    assert e.value.status == 3


@pytest.mark.parametrize("dtype", DTYPES)
def test_mobilenet_layers_exact(dtype, _lib):
    """Every MobileNet-v1 depthwise layer shape (Table III) at batch 2,
    the exact launch configurations bench.py uses (planner picks per shape)."""
    import synth
    amax = 2 if dtype == "bf16" else 3
    for L in synth.mobilenet_v1_dw(2):
        check_all(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout=NCHW, dtype=dtype, kind="int", amax=amax)


def test_mobilenet_layers_random_fp32(_lib):
    import synth
    for L in synth.mobilenet_v1_dw(2):
        check_all(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout=NCHW, dtype="f32", kind="unif")


# configs[2]: MobileNet-v1 width multipliers x resolutions (Table V).
# Plane sizes 4..112 and channel counts 8..768 hit planner branches the alpha 1.0 / 224 stack never does.
CFG3 = [(a, r) for a in (0.25, 0.5, 0.75) for r in (128, 160, 192, 224)]


@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("alpha,res", CFG3)
def test_cfg3_width_resolution_stack(alpha, res, layout, dtype, kind, _lib):
    """All 13 depthwise layers of every alpha x R variant at batch 2, both layouts, both dtypes: every
    output element against the oracle (bitwise on {-2..2} integers, R2/R3 on U[-1,1])."""
    import synth
    for L in synth.mobilenet_v1_dw(2, alpha=alpha, resolution=res):
        check_all(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout=layout, dtype=dtype, kind=kind, amax=2, seed=3)


# configs[3] stress shapes at batch 2 (every element; the bench-size versions sample, test_gpu_fullsize.py)
CFG4_N2 = [(2, 128, 56, 56, 2, 3, 1, 1), (2, 128, 56, 56, 4, 3, 1, 1), (2, 128, 56, 56, 1, 5, 1, 2),
           (2, 128, 56, 56, 1, 7, 1, 3), (2, 512, 56, 56, 1, 3, 2, 1), (2, 512, 56, 56, 1, 5, 2, 2),
           (2, 512, 56, 56, 1, 7, 2, 3)]


@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("shape", CFG4_N2)
def test_cfg4_stress_shapes(shape, layout, dtype, kind, _lib):
    check_all(*shape, layout=layout, dtype=dtype, kind=kind, amax=1, seed=4)


# NHWC fast path (nhwc.cu): m = 1, 3x3, pad 1, C % 4 == 0 -- ragged tiles, several
# channel-vector counts (grid-stride weight reuse, CV not dividing 256), s = 1, 2.
NHWC_FAST = [
    (2, 8, 16, 16, 1, 3, 1, 1),
    (3, 12, 13, 11, 1, 3, 1, 1),    # CV = 3, ragged TH x TW tiles
    (2, 24, 15, 9, 1, 3, 2, 1),     # CV = 6, stride 2, odd sizes
    (1, 1028, 7, 7, 1, 3, 1, 1),    # CV = 257 > 256: two channel groups in bwd_filter
    (2, 64, 28, 28, 1, 3, 2, 1),
    (2, 96, 30, 30, 1, 3, 1, 1),    # TMA tiles: ragged 16-wide columns, 7/8-row tiles
    (2, 96, 30, 34, 1, 3, 2, 1),    # TMA stride 2: odd output widths, ragged tiles
    (1, 256, 9, 21, 1, 3, 2, 1),    # TMA bwd_data polyphase: odd H, W (dx rows/columns past the last dy)
]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", NHWC_FAST)
def test_nhwc_fast_path(shape, dtype, _lib):
    import paper_1803_09926_b200.ops as ops
    n, c, h, w, m, k, s, p = shape
    d = ops.make_desc(n, c, h, w, m, k, s, p, NHWC, 0 if dtype == "f32" else 1)
    for pas in (0, 1):
        assert ops.dwconv_plan(d, pas)["variant_name"] in ("nhwc_tile", "nhwc_tma"), (shape, pas)
    assert ops.dwconv_plan(d, 2)["variant_name"] in ("nhwc_tile", "nhwc_tma"), shape
    check_all(*shape, layout=NHWC, dtype=dtype, kind="unif")
    check_all(*shape, layout=NHWC, dtype=dtype, kind="int", amax=2 if dtype == "bf16" else 3)


@pytest.mark.parametrize("dtype", DTYPES)
def test_mobilenet_layers_exact_nhwc(dtype, _lib):
    """All 13 MobileNet-v1 layers in NHWC (configs[2] layout) through the NHWC kernels."""
    import synth
    import paper_1803_09926_b200.ops as ops
    amax = 2 if dtype == "bf16" else 3
    for L in synth.mobilenet_v1_dw(2):
        d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NHWC, 0 if dtype == "f32" else 1)
        assert ops.dwconv_plan(d, 2)["variant_name"] in ("nhwc_tile", "nhwc_tma")
        assert 0 < ops.dwconv_plan(d, 2)["max_chain"] <= 160
        check_all(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout=NHWC, dtype=dtype, kind="int", amax=amax)


# Fused backward (dwconv_bwd): NCHW 3x3 s=1 m=1 shapes take one
# kernel that produces dx and dw from a single pass over x and dy.
FUSED_SHAPES = [
    (2, 8, 16, 16, 1, 3, 1, 1),
    (3, 5, 13, 11, 1, 3, 1, 1),     # ragged, W not a multiple of 4
    (2, 3, 80, 80, 1, 3, 1, 1),     # band mode: dy halo rows staged per band
    (3, 40, 7, 7, 1, 3, 1, 1),
    (2, 6, 14, 14, 1, 3, 1, 1),
]


def _run_fused(inp, s, p, dtype):
    import paper_1803_09926_b200 as dwl
    x = to_dev(inp["x"], NCHW, dtype)
    w = to_dev(inp["w"], NCHW, dtype)
    dy = to_dev(inp["dy"], NCHW, dtype)
    dx, dw = dwl.bwd(x, dy, w, s, p)
    dx2 = dwl.bwd_data(dy, w, x.shape, s, p)
    torch.cuda.synchronize()
    return dx, dw, dx2


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", FUSED_SHAPES)
def test_fused_backward(shape, dtype, _lib):
    import paper_1803_09926_b200.ops as ops
    from gpu_util import to_np
    n, c, h, w, m, k, s, p = shape
    d = ops.make_desc(n, c, h, w, m, k, s, p, NCHW, 0 if dtype == "f32" else 1)
    # fused kernel for fp32; bf16 takes the two-call path (measured faster)
    assert ops.dwconv_plan(d, 3)["variant_name"] == ("nchw_chunk" if dtype == "f32" else "none"), shape
    if dtype == "f32":
        assert ops.dwconv_plan(d, 3)["max_chain"] <= 160
    for kind in ("unif", "int"):
        inp = make_inputs(*shape, kind=kind, dtype=dtype, amax=2 if dtype == "bf16" else 3)
        dx, dwv, dx_two = _run_fused(inp, s, p, dtype)
        _, (rdx, adx), (rdw, adw) = run_oracle(inp, s, p)
        check_close(to_np(dx), rdx, adx, dtype, "fused dx", kind == "int")
        check_close(to_np(dwv), rdw, adw, "f32", "fused dw", kind == "int")
        # dx comes from the same stencil arithmetic as dwconv_bwd_data (tap order per output)
        assert torch.equal(dx, dx_two), shape


def test_fused_backward_fallback_and_layers(_lib):
    """Shapes without a fused kernel fall back to the two calls; the MobileNet
    stride-1 layers all fuse (batch 2, exact on integers)."""
    import synth
    import paper_1803_09926_b200.ops as ops
    from gpu_util import to_np
    d = ops.make_desc(2, 4, 9, 9, 2, 3, 1, 1, NCHW, 0)  # m = 2: fallback
    info = ops.dwconv_plan(d, 3)
    assert info["variant_name"] == "none" and info["launches"] == 2
    inp = make_inputs(2, 4, 9, 9, 2, 3, 1, 1, kind="int")
    dx, dwv, _ = _run_fused(inp, 1, 1, "f32")
    _, (rdx, adx), (rdw, adw) = run_oracle(inp, 1, 1)
    check_close(to_np(dx), rdx, adx, "f32", "fallback dx", True)
    check_close(to_np(dwv), rdw, adw, "f32", "fallback dw", True)
    for L in synth.mobilenet_v1_dw(2):
        if L.s != 1:
            continue
        d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NCHW, 0)
        assert ops.dwconv_plan(d, 3)["variant_name"] == "nchw_chunk", L
        inp = make_inputs(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, kind="int")
        dx, dwv, _ = _run_fused(inp, L.s, L.p, "f32")
        _, (rdx, adx), (rdw, adw) = run_oracle(inp, L.s, L.p)
        check_close(to_np(dx), rdx, adx, "f32", "fused dx", True)
        check_close(to_np(dwv), rdw, adw, "f32", "fused dw", True)


# the paper's block-diagonal GEMM on tcgen05 (NHWC bf16, stride 1, K = 3/5/7, C % 64 == 0),
# every group size S the library offers, fwd and bwd_data, against the oracle on every element.
BDMMA_SHAPES = [
    (2, 64, 16, 16, 1, 3, 1, 1),     # one tile column, ragged rows
    (2, 128, 37, 45, 1, 3, 1, 1),    # ragged tiles both ways, two channel blocks
    (1, 64, 28, 28, 1, 5, 1, 2),
    (2, 128, 23, 61, 1, 7, 1, 3),    # three tile columns (TW = 26), ragged
    (1, 64, 9, 9, 1, 7, 1, 2),       # padding below (K-1)/2
    (3, 192, 14, 14, 1, 5, 1, 2),
]


@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("shape", BDMMA_SHAPES)
def test_bdmma_candidates(shape, kind, _lib):
    from paper_1803_09926_b200 import ops
    from paper_1803_09926_b200._lib import BF16
    N, C, H, W, m, K, s, p = shape
    inp = make_inputs(N, C, H, W, m, K, s, p, kind=kind, dtype="bf16", amax=1, seed=5)
    (y, ay), (dx, adx), _ = run_oracle(inp, s, p)
    d = ops.make_desc(N, C, H, W, m, K, s, p, NHWC, BF16)
    x = to_dev(inp["x"], NHWC, "bf16")
    w = to_dev(inp["w"], NHWC, "bf16")
    dy = to_dev(inp["dy"], NHWC, "bf16")
    seen = 0
    for pas, out, ref, ab in ((0, torch.empty_like(dy), y, ay), (1, torch.empty_like(x), dx, adx)):
        cands = ops.dwconv_plan_candidates(d, pas)
        idx = [i for i, c in enumerate(cands) if c["variant_name"] == "nhwc_bdmma"]
        assert idx, f"no block-diagonal MMA candidate for {shape} pass {pas}"
        try:
            for i in idx:
                ops.dwconv_plan_select(d, pas, i)
                out.fill_(float("nan"))
                if pas == 0:
                    ops.dwconv_fwd(d, x, w, out)
                else:
                    ops.dwconv_bwd_data(d, dy, w, out)
                torch.cuda.synchronize()
                got = out.float().contiguous().cpu().numpy().astype(np.float64)
                check_close(got, ref, ab, "bf16", f"bdmma S={cands[i]['planes_per_chunk']} CB={cands[i]['rows_per_band']} pass {pas}",
                            kind == "int")
                seen += 1
        finally:
            ops.dwconv_plan_select(d, pas, -1)
    assert seen >= 4


# NHWC general kernels (nhwc_gen.cu): K = 3/5/7, stride 1/2, m = 1/2/4, C % 4 == 0, pad (K-1)/2 -- the shapes
# the 3x3 / m = 1 NHWC families do not take.  Ragged tiles, odd sizes, one and several channel blocks.
NHWC_GEN_SHAPES = [
    (2, 8, 13, 11, 2, 3, 1, 1),
    (2, 12, 9, 10, 4, 3, 1, 1),
    (1, 16, 15, 17, 1, 5, 1, 2),
    (2, 8, 14, 13, 1, 7, 1, 3),
    (2, 140, 11, 9, 1, 5, 2, 2),     # 35 channel vectors: two channel blocks, ragged
    (1, 8, 17, 15, 1, 7, 2, 3),
    (2, 4, 12, 12, 2, 5, 2, 2),
    (3, 8, 7, 9, 4, 3, 2, 1),
    (2, 4, 8, 8, 2, 7, 1, 3),
    # channel counts that take the TMA-staged bwd_filter (C % 16 fp32 / % 32 bf16), ragged bands and columns
    (2, 32, 13, 11, 2, 3, 1, 1),
    (2, 64, 15, 17, 1, 5, 1, 2),
    (1, 32, 14, 13, 1, 7, 2, 3),
    (3, 64, 9, 10, 4, 3, 2, 1),
    (1, 96, 30, 29, 1, 7, 1, 3),
]


@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("shape", NHWC_GEN_SHAPES)
def test_nhwc_gen_kernels(shape, dtype, kind, _lib):
    from paper_1803_09926_b200 import ops
    from paper_1803_09926_b200._lib import BF16, F32
    N, C, H, W, m, K, s, p = shape
    d = ops.make_desc(N, C, H, W, m, K, s, p, NHWC, F32 if dtype == "f32" else BF16)
    for pas in (0, 1, 2):
        assert ops.dwconv_plan(d, pas)["variant_name"] == "nhwc_gen", (shape, pas)
    check_all(*shape, layout=NHWC, dtype=dtype, kind=kind, amax=1, seed=6)

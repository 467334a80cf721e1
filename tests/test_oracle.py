"""Pins of the CPU oracle to things other than itself.

Everything here runs on CPU (``-m "not gpu"``).  The oracle is checked against:
  P1  Eqs. 1-3: a STANDARD (dense) convolution with the masked block-diagonal
      weight equals the depthwise result;
  P2  Eq. 4: the masked dense weight gradient keeps exactly the depthwise dw
      (P:295-301);
  P3  adjoint identities <dy, fwd(x)> = <bwd_data(dy), x> = <bwd_filter(x,dy), w>;
  P4  central finite differences (fp64, h=1e-4);
  P5  hand-worked closed forms (tests/golden/closed_forms.json);
  P7  torch CPU float64 conv2d(groups=C) and its two gradients (a library routine);
  P8  linearity and batch additivity of dw (the data-parallel identity).
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F
from hypothesis import given, settings, strategies as st

import oracle
import synth

NCHW, NHWC = oracle.NCHW, oracle.NHWC

SPECS = [  # (N, C, H, W, m, K, s, p): SURVEY §8(c) c.4 shapes + extras
    (2, 3, 7, 5, 2, 3, 2, 1),
    (1, 4, 6, 6, 1, 5, 1, 2),
    (2, 2, 9, 8, 3, 3, 2, 0),
    (1, 2, 5, 5, 1, 1, 1, 0),
    (2, 8, 16, 16, 1, 3, 1, 1),
    (1, 3, 11, 7, 1, 7, 1, 3),
    (2, 2, 10, 9, 2, 3, 3, 1),
]


def _ints(seed, shape, a=3):
    return synth.integers(seed, shape, a).astype(np.float64)


def _unif(seed, shape):
    return synth.uniform(seed, shape).astype(np.float64)


def _data(spec, gen):
    N, C, H, W, m, K, s, p = spec
    Ho = (H + 2 * p - K) // s + 1
    Wo = (W + 2 * p - K) // s + 1
    x = gen(11, (N, C, H, W))
    w = gen(12, (C * m, K, K))
    dy = gen(13, (N, C * m, Ho, Wo))
    return x, w, dy


def _to_layout(a, layout):
    return a if layout == NCHW else synth.nchw_to_nhwc(a)


def _from_layout(a, layout):
    return a if layout == NCHW else synth.nhwc_to_nchw(a)


# ---------------------------------------------------------------- P1 / P2
@pytest.mark.parametrize("spec", SPECS)
def test_p1_diagonal_refactorization_eq1_to_eq3(spec):
    N, C, H, W, m, K, s, p = spec
    x, w, _ = _data(spec, _ints)
    wd = oracle.dense_weights(w, C)                    # Eq. 1 (generalised to m)
    A = oracle.mask(C, m, K, K)                        # Eq. 2
    w_hat = oracle.hadamard(wd, A)                     # Eq. 3, W^ = W (.) A
    z_dense = oracle.dense_fwd(x, w_hat, s, p)         # Eq. 3, Z = W^ (x) X
    y, _ = oracle.fwd(x, w, s, p)
    assert np.array_equal(z_dense, y)
    # the block-diagonal structure itself: every off-diagonal block is zero
    for o in range(C * m):
        for ci in range(C):
            if ci != o // m:
                assert not w_hat[o, ci].any()
            else:
                assert np.array_equal(w_hat[o, ci], w[o])


@pytest.mark.parametrize("spec", SPECS)
def test_p2_masked_weight_gradient_eq4(spec):
    N, C, H, W, m, K, s, p = spec
    x, w, dy = _data(spec, _ints)
    A = oracle.mask(C, m, K, K)
    G = oracle.dense_bwd_filter(x, dy, (C * m, C, K, K), s, p)   # dL/dW^
    masked = oracle.hadamard(G, A)                               # Eq. 4
    dw, _ = oracle.bwd_filter(x, dy, w.shape, s, p)
    for o in range(C * m):
        for ci in range(C):
            if ci == o // m:
                assert np.array_equal(masked[o, ci], dw[o])
            else:
                assert not masked[o, ci].any()
    if C > 1:  # the mask is doing real work: the unmasked gradient is not block-diagonal
        off = G * (1.0 - A)
        assert np.abs(off).sum() > 0
    # the dense input gradient through W^ equals the depthwise input gradient
    w_hat = oracle.hadamard(oracle.dense_weights(w, C), A)
    dx_dense = oracle.dense_bwd_data(dy, w_hat, x.shape, s, p)
    dx, _ = oracle.bwd_data(dy, w, x.shape, s, p)
    assert np.array_equal(dx_dense, dx)


# ---------------------------------------------------------------- P3
@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("spec", SPECS)
def test_p3_adjoint_identities(spec, layout):
    N, C, H, W, m, K, s, p = spec
    for gen, exact in ((_ints, True), (_unif, False)):
        x, w, dy = _data(spec, gen)
        xl, dyl = _to_layout(x, layout), _to_layout(dy, layout)
        y, _ = oracle.fwd(xl, w, s, p, layout)
        dx, _ = oracle.bwd_data(dyl, w, xl.shape, s, p, layout)
        dw, _ = oracle.bwd_filter(xl, dyl, w.shape, s, p, layout)
        a = float(np.sum(dyl * y))
        b = float(np.sum(dx * xl))
        c = float(np.sum(dw * w))
        if exact:
            assert a == b == c
        else:
            scale = float(np.sum(np.abs(dyl) * np.abs(y))) + 1.0
            assert abs(a - b) <= 1e-12 * scale and abs(a - c) <= 1e-12 * scale


# ---------------------------------------------------------------- P4
@pytest.mark.parametrize("spec", [SPECS[0], SPECS[1], SPECS[6]])
def test_p4_finite_differences(spec):
    """L(x, w) = <dy, fwd(x; w)>; dL/dx = bwd_data(dy), dL/dw = bwd_filter(x, dy)."""
    N, C, H, W, m, K, s, p = spec
    x, w, dy = _data(spec, _unif)
    h = 1e-4

    def L(xx, ww):
        return float(np.sum(dy * oracle.fwd(xx, ww, s, p)[0]))

    dx, _ = oracle.bwd_data(dy, w, x.shape, s, p)
    dw, _ = oracle.bwd_filter(x, dy, w.shape, s, p)
    worst = 0.0
    for idx in np.ndindex(*x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        num = (L(xp, w) - L(xm, w)) / (2 * h)
        worst = max(worst, abs(num - dx[idx]) / max(abs(num), abs(dx[idx]), 1e-12))
    for idx in np.ndindex(*w.shape):
        wp, wm = w.copy(), w.copy()
        wp[idx] += h
        wm[idx] -= h
        num = (L(x, wp) - L(x, wm)) / (2 * h)
        worst = max(worst, abs(num - dw[idx]) / max(abs(num), abs(dw[idx]), 1e-12))
    assert worst <= 1e-6


# ---------------------------------------------------------------- P5
def _closed_cases(golden_dir):
    with open(os.path.join(golden_dir, "closed_forms.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("layout", [NCHW, NHWC])
def test_p5_closed_forms(golden_dir, layout):
    for case in _closed_cases(golden_dir):
        N, C, H, W, m, K, s, p = (case[k] for k in ("n", "c", "h", "w", "m", "k", "s", "p"))
        Ho, Wo = (H + 2 * p - K) // s + 1, (W + 2 * p - K) // s + 1
        x = np.ones((N, C, H, W))
        w = np.ones((C * m, K, K))
        dy = np.ones((N, C * m, Ho, Wo))
        xl, dyl = _to_layout(x, layout), _to_layout(dy, layout)
        if case["pass"] == "fwd":
            y = _from_layout(oracle.fwd(xl, w, s, p, layout)[0], layout)
            assert np.array_equal(y[0, 0], np.array(case["expect"], dtype=float)), case["name"]
        elif case["pass"] == "bwd_filter":
            dw = oracle.bwd_filter(xl, dyl, w.shape, s, p, layout)[0]
            if "expect" in case:
                for o in range(C * m):
                    assert np.array_equal(dw[o], np.array(case["expect"], dtype=float)), case["name"]
            else:
                assert np.all(dw == case["expect_all"]), case["name"]
        else:
            dx = _from_layout(oracle.bwd_data(dyl, w, xl.shape, s, p, layout)[0], layout)
            cov = np.array(case["cov"], dtype=float)
            assert np.array_equal(dx[0, 0], m * np.outer(cov, cov)), case["name"]


def test_p5_delta_kernel_identity_and_zero_kernel():
    x = _unif(5, (2, 3, 6, 7))
    dy = _unif(6, (2, 3, 6, 7))
    w = np.zeros((3, 3, 3))
    w[:, 1, 1] = 1.0
    assert np.array_equal(oracle.fwd(x, w, 1, 1)[0], x)
    assert np.array_equal(oracle.bwd_data(dy, w, x.shape, 1, 1)[0], dy)
    z = np.zeros((3, 3, 3))
    assert not oracle.fwd(x, z, 1, 1)[0].any()
    assert not oracle.bwd_data(dy, z, x.shape, 1, 1)[0].any()


def test_p5_k1_is_scaling():
    x = _unif(7, (2, 4, 5, 3))
    dy = _unif(8, (2, 4, 5, 3))
    w = _unif(9, (4, 1, 1))
    y = oracle.fwd(x, w, 1, 0)[0]
    assert np.array_equal(y, x * w[None, :, :, :].reshape(1, 4, 1, 1))
    dw = oracle.bwd_filter(x, dy, w.shape, 1, 0)[0]
    expect = np.array([np.sum(x[:, c] * dy[:, c]) for c in range(4)])
    assert np.allclose(dw[:, 0, 0], expect, rtol=1e-14, atol=0)


# ---------------------------------------------------------------- P7
def _torch_ref(x, w, dy, C, s, p):
    xt, wt, dyt = (torch.from_numpy(a) for a in (x, w, dy))
    wt4 = wt.reshape(wt.shape[0], 1, wt.shape[1], wt.shape[2])
    y = F.conv2d(xt, wt4, stride=s, padding=p, groups=C)
    dx = torch.nn.grad.conv2d_input(xt.shape, wt4, dyt, stride=s, padding=p, groups=C)
    dw = torch.nn.grad.conv2d_weight(xt, wt4.shape, dyt, stride=s, padding=p, groups=C)
    return y.numpy(), dx.numpy(), dw.numpy().reshape(w.shape)


def _check_torch(spec, gen, layout):
    N, C, H, W, m, K, s, p = spec
    x, w, dy = _data(spec, gen)
    ty, tdx, tdw = _torch_ref(x, w, dy, C, s, p)
    xl, dyl = _to_layout(x, layout), _to_layout(dy, layout)
    y, ay = oracle.fwd(xl, w, s, p, layout)
    dx, adx = oracle.bwd_data(dyl, w, xl.shape, s, p, layout)
    dw, adw = oracle.bwd_filter(xl, dyl, w.shape, s, p, layout)
    y, ay, dx, adx = (_from_layout(a, layout) for a in (y, ay, dx, adx))
    if gen is _ints:
        assert np.array_equal(y, ty) and np.array_equal(dx, tdx) and np.array_equal(dw, tdw)
    else:  # both are double sums; differ only by summation order
        for a, b, s_ in ((y, ty, ay), (dx, tdx, adx), (dw, tdw, adw)):
            assert np.all(np.abs(a - b) <= 1e-13 * s_ + 1e-300)
    # the reported sum|terms| really bounds the value
    assert np.all(np.abs(y) <= ay + 1e-12) and np.all(np.abs(dw) <= adw + 1e-12)


@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("spec", SPECS)
def test_p7_torch_cpu_float64(spec, layout):
    _check_torch(spec, _ints, layout)
    _check_torch(spec, _unif, layout)


@settings(max_examples=60, deadline=None)
@given(N=st.integers(1, 2), C=st.integers(1, 6), H=st.integers(1, 9), W=st.integers(1, 9),
       m=st.integers(1, 3), K=st.sampled_from([1, 2, 3, 5]), s=st.integers(1, 3),
       p=st.integers(0, 4), layout=st.sampled_from([NCHW, NHWC]))
def test_p7_property_random_specs(N, C, H, W, m, K, s, p, layout):
    p = min(p, K - 1)
    if H + 2 * p < K or W + 2 * p < K:
        return
    _check_torch((N, C, H, W, m, K, s, p), _ints, layout)


# ---------------------------------------------------------------- P7b: the tolerance basis
# Every float parity tolerance (R11/R13) is scaled by the oracle's per-element
# sum|terms|.  The terms are products of two inputs, so sum|terms| is the same
# convolution applied to |x|, |w| (fwd), |dy|, |w| (bwd_data), |x|, |dy|
# (bwd_filter) over the same in-bounds taps: torch's fp64 conv2d of the absolute
# values computes it independently.  An inflated (out-of-range taps, wrong j
# loop) or deflated sum fails here; on integers the match is bitwise.
def _check_abs_sums(spec, gen, layout):
    N, C, H, W, m, K, s, p = spec
    x, w, dy = _data(spec, gen)
    ty, tdx, tdw = _torch_ref(np.abs(x), np.abs(w), np.abs(dy), C, s, p)
    xl, dyl = _to_layout(x, layout), _to_layout(dy, layout)
    ay = _from_layout(oracle.fwd(xl, w, s, p, layout)[1], layout)
    adx = _from_layout(oracle.bwd_data(dyl, w, xl.shape, s, p, layout)[1], layout)
    adw = oracle.bwd_filter(xl, dyl, w.shape, s, p, layout)[1]
    for name, a, t in (("ABS_y", ay, ty), ("ABS_dx", adx, tdx), ("ABS_dw", adw, tdw)):
        if gen is _ints:
            assert np.array_equal(a, t), name
        else:
            assert np.all(np.abs(a - t) <= 1e-13 * t + 1e-300), (name, np.max(np.abs(a - t) / (t + 1e-300)))


@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("spec", SPECS)
def test_p7b_abs_sums_equal_conv_of_abs_values(spec, layout):
    _check_abs_sums(spec, _ints, layout)
    _check_abs_sums(spec, _unif, layout)


@settings(max_examples=40, deadline=None)
@given(N=st.integers(1, 2), C=st.integers(1, 5), H=st.integers(1, 9), W=st.integers(1, 9),
       m=st.integers(1, 3), K=st.sampled_from([1, 2, 3, 5, 7]), s=st.integers(1, 3),
       p=st.integers(0, 4), layout=st.sampled_from([NCHW, NHWC]))
def test_p7b_abs_sums_property(N, C, H, W, m, K, s, p, layout):
    p = min(p, K - 1)
    if H + 2 * p < K or W + 2 * p < K:
        return
    _check_abs_sums((N, C, H, W, m, K, s, p), _ints, layout)
    _check_abs_sums((N, C, H, W, m, K, s, p), _unif, layout)


def test_rectangular_kernel_stride_pad_against_torch():
    x, w = _ints(1, (2, 3, 9, 11)), _ints(2, (6, 3, 5))
    y, _ = oracle.fwd(x, w, (2, 1), (1, 2))
    ty = F.conv2d(torch.from_numpy(x), torch.from_numpy(w).reshape(6, 1, 3, 5),
                  stride=(2, 1), padding=(1, 2), groups=3).numpy()
    assert np.array_equal(y, ty)


# ---------------------------------------------------------------- P8
def test_p8_linearity_and_batch_additivity():
    spec = (4, 3, 8, 8, 2, 3, 2, 1)
    N, C, H, W, m, K, s, p = spec
    x, w, dy = _data(spec, _ints)
    x2 = _ints(21, x.shape)
    y1 = oracle.fwd(x, w, s, p)[0]
    y2 = oracle.fwd(x2, w, s, p)[0]
    y12 = oracle.fwd(3 * x - 2 * x2, w, s, p)[0]
    assert np.array_equal(y12, 3 * y1 - 2 * y2)
    full = oracle.bwd_filter(x, dy, w.shape, s, p)[0]
    parts = sum(oracle.bwd_filter(x[r:r + 1], dy[r:r + 1], w.shape, s, p)[0] for r in range(N))
    assert np.array_equal(full, parts)
    halves = (oracle.bwd_filter(x[:2], dy[:2], w.shape, s, p)[0] +
              oracle.bwd_filter(x[2:], dy[2:], w.shape, s, p)[0])
    assert np.array_equal(full, halves)


def test_out_size_and_kernel_exceeds_input():
    assert oracle.out_size(112, 3, 2, 1) == 56
    assert oracle.out_size(7, 3, 1, 1) == 7
    assert oracle.out_size(2, 5, 1, 0) is None
    with pytest.raises(ValueError):
        oracle.fwd(np.zeros((1, 1, 2, 2)), np.zeros((1, 5, 5)), 1, 0)


# ---------------------------------------------------------------- storage rounding
def test_round_f32_matches_numpy_cast():
    v = _unif(3, (1000,)) * 1e3 + np.ldexp(_unif(4, (1000,)), -30)
    assert np.array_equal(oracle.round_to(v, "f32"), v.astype(np.float32).astype(np.float64))


def test_round_bf16_single_rounding():
    one = 1.0
    cases = [
        (one + 2.0 ** -8, one),                        # exact tie -> even (mantissa 0)
        (one + 3 * 2.0 ** -8, one + 2.0 ** -6),        # exact tie -> even (mantissa 2)
        (one + 2.0 ** -8 + 2.0 ** -30, one + 2.0 ** -7),  # above the tie: a double rounding via fp32 would give 1.0
        (-(one + 2.0 ** -8 + 2.0 ** -30), -(one + 2.0 ** -7)),
        (0.0, 0.0),
        (3.0, 3.0),
        (2.0 ** -130, 2.0 ** -130),                     # bf16 subnormal grid 2^-133
        (2.0 ** -134, 0.0),                             # half of the smallest subnormal: tie -> 0
        (3.0 * 2.0 ** -134, 2.0 ** -132),               # 1.5 ulp -> even (2 ulp)
        (2.0 ** 128, float("inf")),
        (255.0 * 2.0 ** 120, 255.0 * 2.0 ** 120),       # largest finite bf16
    ]
    got = oracle.round_to(np.array([c[0] for c in cases]), "bf16")
    assert np.array_equal(got, np.array([c[1] for c in cases]))
    # agrees with the fp32->bf16 RNE of synth on fp32-representable inputs
    v = synth.uniform(9, (4096,)).astype(np.float64) * 7.0
    via_f32 = synth._bf16_round_f32(v.astype(np.float32)).astype(np.float64)
    assert np.array_equal(oracle.round_to(v, "bf16"), via_f32)


@pytest.mark.parametrize("layout", [NCHW, NHWC])
@pytest.mark.parametrize("spec", SPECS)
def test_threaded_oracle_bitwise_equals_sequential(spec, layout):
    """The all-cores CPU baseline splits only the outer loops over OpenMP threads: every
    output element (value and sum|terms|) must be bitwise equal to the sequential oracle's."""
    N, C, H, W, m, K, s, p = spec
    x, w, dy = (_to_layout(a, layout) if a.ndim == 4 else a for a in _data(spec, _unif))
    shp = x.shape  # physical shape in the layout (the oracle's convention)
    runs = []
    for t in (1, 4):
        oracle.set_threads(t)
        try:
            runs.append([oracle.fwd(x, w, s, p, layout=layout), oracle.bwd_data(dy, w, shp, s, p, layout=layout),
                         oracle.bwd_filter(x, dy, w.shape, s, p, layout=layout)])
        finally:
            oracle.set_threads(1)
    for r1, r4 in zip(*runs):
        for a, b in zip(r1, r4):
            assert np.array_equal(a, b)

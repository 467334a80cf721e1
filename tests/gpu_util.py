"""Shared helpers for the GPU parity tests: run the CUDA path and the oracle on the
same seeded inputs and compare element by element."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

NCHW, NHWC = 0, 1


def make_inputs(N, C, H, W, m, K, s, p, kind="unif", dtype="f32", amax=3, seed=0):
    Ho, Wo = (H + 2 * p - K) // s + 1, (W + 2 * p - K) // s + 1
    shapes = {"x": (N, C, H, W), "w": (C * m, K, K), "dy": (N, C * m, Ho, Wo)}
    out = {}
    for i, (name, shp) in enumerate(shapes.items()):
        if kind == "int":
            out[name] = synth.integers(seed * 10 + i + 1, shp, amax)
        else:
            out[name] = synth.uniform(seed * 10 + i + 1, shp, dtype)
    return out


def to_dev(a: np.ndarray, layout: int, dtype: str) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    t = t.to(torch.bfloat16) if dtype == "bf16" else t
    t = t.cuda()
    if layout == NHWC and t.dim() == 4:
        t = t.contiguous(memory_format=torch.channels_last)
    return t


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.float().contiguous().cpu().numpy().astype(np.float64)


def run_gpu(inp, s, p, layout, dtype):
    import paper_1803_09926_b200 as dw
    x = to_dev(inp["x"], layout, dtype)
    w = to_dev(inp["w"], layout, dtype)
    dy = to_dev(inp["dy"], layout, dtype)
    y = dw.fwd(x, w, s, p)
    dx = dw.bwd_data(dy, w, x.shape, s, p)
    dwt = dw.bwd_filter(x, dy, w.shape, s, p)
    torch.cuda.synchronize()
    return to_np(y), to_np(dx), to_np(dwt)


def run_oracle(inp, s, p):
    x, w, dy = (inp[k].astype(np.float64) for k in ("x", "w", "dy"))
    y, ay = oracle.fwd(x, w, s, p)
    dx, adx = oracle.bwd_data(dy, w, x.shape, s, p)
    dwv, adw = oracle.bwd_filter(x, dy, w.shape, s, p)
    return (y, ay), (dx, adx), (dwv, adw)


def check_close(gpu, ref, absum, dtype, what, exact=False):
    """Parity contract: exact (integers), R2 fp32, R3 bf16 (reading R11/R18)."""
    if exact:
        rr = oracle.round_to(ref, dtype)
        bad = np.argwhere(gpu != rr)
        assert bad.size == 0, f"{what}: {len(bad)} mismatches, first {bad[0]}: gpu {gpu[tuple(bad[0])]} ref {rr[tuple(bad[0])]}"
        return
    tol = 1e-5 * absum
    if dtype == "bf16":
        tol = tol + 1e-2 * np.abs(ref)
    err = np.abs(gpu - ref)
    bad = err > tol
    assert not bad.any(), (f"{what}: {int(bad.sum())} elements outside tolerance; worst err "
                           f"{err.max():.3e} at {np.unravel_index(np.argmax(err - tol), err.shape)}")
    zero = absum == 0
    assert np.all(gpu[zero] == 0), f"{what}: nonzero where every term is zero"


def check_all(N, C, H, W, m, K, s, p, layout, dtype, kind, seed=0, amax=3):
    inp = make_inputs(N, C, H, W, m, K, s, p, kind=kind, dtype=dtype, amax=amax, seed=seed)
    gy, gdx, gdw = run_gpu(inp, s, p, layout, dtype)
    (y, ay), (dx, adx), (dwv, adw) = run_oracle(inp, s, p)
    exact = kind == "int"
    check_close(gy, y, ay, dtype, "fwd", exact)
    check_close(gdx, dx, adx, dtype, "bwd_data", exact)
    check_close(gdw, dwv, adw, "f32", "bwd_filter", exact)

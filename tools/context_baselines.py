"""Same-box context baselines -- NOT targets, NOT the product path.

Times, on the same B200 and the same MobileNet-v1 depthwise stack as bench.py:

* cuDNN depthwise: torch F.conv2d(groups=C) forward and the cuDNN input / weight
  gradients (torch.nn.grad.conv2d_input / conv2d_weight);
* the paper's diagonalwise refactorization (§III, Eqs. 1-4)
  executed the way the paper does it -- the depthwise weights scattered into
  block-diagonal dense weights of group size S (Eq. 1 with mask A, Eq. 2) and a
  standard grouped convolution (groups = C / S) run by cuDNN; the weight gradient
  is the dense grouped gradient (Eq. 4 then keeps its diagonal);
* this repo's kernels (library calls, planner defaults or --tune).

Per layer and pass: mean us of back-to-back launches (CUDA events, eager, inputs
rotated over >= 2x L2 of copies).  Prints one JSON object; `--md FILE` writes a
markdown table.  Example:  python tools/context_baselines.py --md profiles/r1/context_baselines.md
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import synth  # noqa: E402
from paper_1803_09926_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--groups", default="8,32", help="diagonalwise group sizes S (channels per dense block)")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tune", action="store_true", help="measured plan selection for this repo's kernels")
ap.add_argument("--md", default="")
a = ap.parse_args()
dev = torch.device("cuda")
dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
eb = 4 if a.dtype == "f32" else 2
torch.backends.cudnn.benchmark = True
l2 = torch.cuda.get_device_properties(dev).L2_cache_size


def timed(fn_sets, reps):
    for f in fn_sets:
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        for f in fn_sets:
            f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * len(fn_sets))


res = {"batch": a.batch, "dtype": a.dtype, "layers": {}}
for L in synth.mobilenet_v1_dw(a.batch):
    xb = L.x_elems() * eb
    yb = L.y_elems() * eb
    nsets = int(max(2, min(8, -(-2 * l2 // (2 * (xb + yb))))))
    sets = [(torch.randn(L.n, L.c, L.h, L.w, device=dev, dtype=dt), torch.randn(L.n, L.c, L.ho, L.wo, device=dev, dtype=dt))
            for _ in range(nsets)]
    w = torch.randn(L.c, 1, 3, 3, device=dev, dtype=dt)
    row = {}
    # cuDNN depthwise
    row["cudnn_dw"] = {
        "fwd": timed([lambda s=s: F.conv2d(s[0], w, None, L.s, 1, 1, L.c) for s in sets], a.reps),
        "bwd_data": timed([lambda s=s: torch.nn.grad.conv2d_input(s[0].shape, w, s[1], L.s, 1, 1, L.c) for s in sets],
                          a.reps),
        "bwd_filter": timed([lambda s=s: torch.nn.grad.conv2d_weight(s[0], w.shape, s[1], L.s, 1, 1, L.c)
                             for s in sets], a.reps)}
    # diagonalwise refactorization (block-diagonal dense groups of S channels)
    for S in [int(v) for v in a.groups.split(",")]:
        if L.c % S:
            continue
        G = L.c // S
        wd = torch.zeros(L.c, S, 3, 3, device=dev, dtype=dt)  # Eq. 1-2: W_hat = W (.) A, block diagonal
        idx = torch.arange(L.c, device=dev)
        wd[idx, idx % S] = w[:, 0]
        row[f"diag_S{S}"] = {
            "fwd": timed([lambda s=s: F.conv2d(s[0], wd, None, L.s, 1, 1, G) for s in sets], a.reps),
            "bwd_data": timed([lambda s=s: torch.nn.grad.conv2d_input(s[0].shape, wd, s[1], L.s, 1, 1, G)
                               for s in sets], a.reps),
            "bwd_filter": timed([lambda s=s: torch.nn.grad.conv2d_weight(s[0], wd.shape, s[1], L.s, 1, 1, G)
                                 for s in sets], a.reps)}
    # this repo
    d = ops.make_desc(L.n, L.c, L.h, L.w, 1, 3, L.s, 1, 0, 0 if a.dtype == "f32" else 1)
    wk = w.reshape(L.c, 3, 3).contiguous()
    if a.tune:
        from paper_1803_09926_b200 import tune
        tune.tune_layer(d, sets[0][0], sets[0][1], wk)
    ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device=dev)
    y = torch.empty(L.n, L.c, L.ho, L.wo, device=dev, dtype=dt)
    dx = torch.empty(L.n, L.c, L.h, L.w, device=dev, dtype=dt)
    dwt = torch.empty(L.c, 3, 3, device=dev)
    row["this_repo"] = {
        "fwd": timed([lambda s=s: ops.dwconv_fwd(d, s[0], wk, y) for s in sets], a.reps),
        "bwd_data": timed([lambda s=s: ops.dwconv_bwd_data(d, s[1], wk, dx) for s in sets], a.reps),
        "bwd_filter": timed([lambda s=s: ops.dwconv_bwd_filter(d, s[0], s[1], dwt, ws) for s in sets], a.reps)}
    res["layers"][L.name] = row
    del sets
    torch.cuda.empty_cache()

impls = sorted({k for r in res["layers"].values() for k in r})
res["step_us"] = {k: sum(sum(r[k].values()) for r in res["layers"].values() if k in r) for k in impls}
res["img_s_serial"] = {k: a.batch / (v * 1e-6) for k, v in res["step_us"].items()}
print(json.dumps(res))
if a.md:
    lines = [f"# Same-box context baselines — MobileNet-v1 depthwise stack, batch {a.batch}, {a.dtype}, NCHW, one B200",
             "", "Context only (SURVEY §8(f) NEXT-4), not a target.  Eager back-to-back launches, inputs rotated over",
             ">= 2x L2, mean µs per launch; the step sum is serial (no stream overlap, unlike bench.py).",
             "`diag_S{S}` = the paper's diagonalwise refactorization (block-diagonal dense weights, groups = C/S, cuDNN).", "",
             "| layer | " + " | ".join(f"{k} fwd / bd / bf µs" for k in impls) + " |",
             "|---|" + "---|" * len(impls)]
    for name, r in res["layers"].items():
        cells = []
        for k in impls:
            cells.append(" / ".join(f"{r[k][p]:.1f}" for p in ("fwd", "bwd_data", "bwd_filter")) if k in r else "-")
        lines.append(f"| {name} | " + " | ".join(cells) + " |")
    lines += ["", "| impl | serial step µs | images/s (serial) |", "|---|---|---|"]
    for k in impls:
        lines.append(f"| {k} | {res['step_us'][k]:.0f} | {res['img_s_serial'][k]:.0f} |")
    os.makedirs(os.path.dirname(a.md) or ".", exist_ok=True)
    open(a.md, "w").write("\n".join(lines) + "\n")

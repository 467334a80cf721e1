"""Run one (layer, pass) of the MobileNet-v1 depthwise stack a few times (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1803_09926_b200 as dwl  # noqa: E402
from paper_1803_09926_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="dw2")
ap.add_argument("--pass", dest="pas", default="fwd", choices=["fwd", "bwd_data", "bwd_filter", "all"])
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--alpha", type=float, default=1.0)
ap.add_argument("--res", type=int, default=224)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--layout", default="nchw")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--plan", action="store_true")
ap.add_argument("--plans", default="", help="bench.py --plans file: install this layer's measured selection")
a, _unknown = ap.parse_known_args()  # bench.py args pass through (profile_round.sh)
L = [l for l in synth.mobilenet_v1_dw(a.batch, a.alpha, a.res) if l.name == a.layer][0]
lay = dwl.NCHW if a.layout == "nchw" else dwl.NHWC
dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
mf = torch.channels_last if lay == dwl.NHWC else torch.contiguous_format
d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, lay, 0 if a.dtype == "f32" else 1)
x = torch.randn(L.n, L.c, L.h, L.w, device="cuda").to(dt).contiguous(memory_format=mf)
dy = torch.randn(L.n, L.c * L.m, L.ho, L.wo, device="cuda").to(dt).contiguous(memory_format=mf)
w = torch.randn(L.c * L.m, L.k, L.k, device="cuda").to(dt)
y = torch.empty_like(dy)
dx = torch.empty_like(x)
dw = torch.empty(L.c * L.m, L.k, L.k, device="cuda")
if a.plans and os.path.exists(a.plans):
    import json
    from paper_1803_09926_b200 import tune
    with open(a.plans) as f:
        tune.apply_selection(d, json.load(f).get(a.layer, {}))
ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
if a.plan:
    for p in range(3):
        print(L, p, ops.dwconv_plan(d, p))
for _ in range(a.reps):
    if a.pas in ("fwd", "all"):
        ops.dwconv_fwd(d, x, w, y)
    if a.pas in ("bwd_data", "all"):
        ops.dwconv_bwd_data(d, dy, w, dx)
    if a.pas in ("bwd_filter", "all"):
        ops.dwconv_bwd_filter(d, x, dy, dw, ws)
torch.cuda.synchronize()

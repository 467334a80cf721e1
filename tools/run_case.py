"""Launch one pass of one shape with one candidate plan a few times (for ncu captures).

    python tools/run_case.py --shape 64,128,56,56,1,3,1,1 --dtype bf16 --layout nhwc --pass fwd --cand 15 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_09926_b200 import ops  # noqa: E402
from paper_1803_09926_b200._lib import BF16, F32, NCHW, NHWC  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", required=True)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--layout", default="nhwc")
ap.add_argument("--pass", dest="pas", default="fwd")
ap.add_argument("--cand", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
N, C, H, W, m, K, s, p = (int(v) for v in a.shape.split(","))
lay = NCHW if a.layout == "nchw" else NHWC
d = ops.make_desc(N, C, H, W, m, K, s, p, lay, F32 if a.dtype == "f32" else BF16)
Ho, Wo = ops.output_shape(d)
tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
mf = torch.channels_last if lay == NHWC else torch.contiguous_format
x = torch.randn(N, C, H, W, device="cuda").to(tdt).contiguous(memory_format=mf)
dy = torch.randn(N, C * m, Ho, Wo, device="cuda").to(tdt).contiguous(memory_format=mf)
w = torch.randn(C * m, K, K, device="cuda").to(tdt)
y, dx = torch.empty_like(dy), torch.empty_like(x)
dw = torch.empty(C * m, K, K, device="cuda")
pas = {"fwd": 0, "bwd_data": 1, "bwd_filter": 2}[a.pas]
if a.cand >= 0:
    cands = ops.dwconv_plan_candidates(d, pas)
    ops.dwconv_plan_select(d, pas, a.cand)
    print("candidate", a.cand, cands[a.cand])
ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    if pas == 0:
        ops.dwconv_fwd(d, x, w, y)
    elif pas == 1:
        ops.dwconv_bwd_data(d, dy, w, dx)
    else:
        ops.dwconv_bwd_filter(d, x, dy, dw, ws)
torch.cuda.synchronize()
print("done")

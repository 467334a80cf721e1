"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [--all-candidates]

Cases (batch 2-4 so racecheck finishes): configs[0]; a small-plane layer (14x14, warp-task rings);
a band bwd_filter layer (112x112 / 56x56 NCHW); an NHWC TMA layer (s=1, s=2); a stride-2 polyphase
bwd_data; K=5/7 and m=2 (generic / NHWC paths); bf16.  Each pass of each case runs through the C ABI;
with --all-candidates every candidate plan of the pass runs too (workspace tickets, finalize trees).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1803_09926_b200 import ops  # noqa: E402
from paper_1803_09926_b200._lib import BF16, F32, NCHW, NHWC  # noqa: E402

CASES = [  # name, (N, C, H, W, m, K, s, p), layout, dtype
    ("cfg1", (2, 8, 16, 16, 1, 3, 1, 1), NCHW, "f32"),
    ("small14", (4, 32, 14, 14, 1, 3, 1, 1), NCHW, "f32"),
    ("small7_bf16", (4, 64, 7, 7, 1, 3, 1, 1), NCHW, "bf16"),
    ("band112", (2, 8, 112, 112, 1, 3, 1, 1), NCHW, "f32"),
    # round 3: bf16 interleaved strips, producer-warp bwd_filter, streaming bwd_filter and s2 bwd_data, m = 1 kernels
    ("bf16_112", (2, 32, 112, 112, 1, 3, 1, 1), NCHW, "bf16"),
    ("bf16_112_s2", (2, 32, 112, 112, 1, 3, 2, 1), NCHW, "bf16"),
    # round 3: lane-per-plane kernels (C % 32 == 0)
    ("lane14_bf16", (4, 64, 14, 14, 1, 3, 1, 1), NCHW, "bf16"),
    ("band56_s2", (2, 16, 56, 56, 1, 3, 2, 1), NCHW, "f32"),
    ("nhwc_tma_s1", (2, 64, 28, 28, 1, 3, 1, 1), NHWC, "f32"),
    ("nhwc_tma_s2_bf16", (2, 128, 28, 28, 1, 3, 2, 1), NHWC, "bf16"),
    ("k5", (2, 32, 28, 28, 1, 5, 1, 2), NCHW, "f32"),
    ("k7_nhwc", (2, 32, 28, 28, 1, 7, 1, 3), NHWC, "bf16"),
    ("m2", (2, 16, 28, 28, 2, 3, 1, 1), NHWC, "f32"),
    ("bdmma_k5", (2, 64, 20, 20, 1, 5, 1, 2), NHWC, "bf16"),  # tcgen05 block-diagonal candidates
    ("small14_s2", (4, 32, 14, 14, 1, 3, 2, 1), NCHW, "f32"),  # stride-2 small-plane fwd / bwd_data / bwd_filter
    ("small14_s2_bf16", (2, 64, 14, 14, 1, 3, 2, 1), NCHW, "bf16"),  # 8-plane tasks / 8-channel groups
    ("nhwc_gen_k5", (2, 64, 20, 20, 1, 5, 1, 2), NHWC, "f32"),  # NHWC general kernels, TMA-staged bwd_filter
]


def run(name, shp, layout, dtype, all_cands, skip=()):
    N, C, H, W, m, K, s, p = shp
    d = ops.make_desc(N, C, H, W, m, K, s, p, layout, F32 if dtype == "f32" else BF16)
    Ho, Wo = ops.output_shape(d)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    mf = torch.channels_last if layout == NHWC else torch.contiguous_format
    x = torch.randn(N, C, H, W, device="cuda").to(tdt).contiguous(memory_format=mf)
    dy = torch.randn(N, C * m, Ho, Wo, device="cuda").to(tdt).contiguous(memory_format=mf)
    w = torch.randn(C * m, K, K, device="cuda").to(tdt)
    y = torch.empty_like(dy)
    dx = torch.empty_like(x)
    dw = torch.empty(C * m, K, K, device="cuda")
    for pas in (0, 1, 2):
        cands = ops.dwconv_plan_candidates(d, pas) if all_cands else []
        idxs = [i for i in range(len(cands)) if cands[i]["variant_name"] not in skip] or [None]
        ws = torch.zeros(max([16, ops.dwconv_bwd_filter_workspace_bytes(d)] +
                             [c["workspace_bytes"] for c in cands]), dtype=torch.uint8, device="cuda")
        for i in idxs:
            if i is not None:
                ops.dwconv_plan_select(d, pas, i)
            if pas == 0:
                ops.dwconv_fwd(d, x, w, y)
            elif pas == 1:
                ops.dwconv_bwd_data(d, dy, w, dx)
            else:
                ops.dwconv_bwd_filter(d, x, dy, dw, ws)
        if cands:
            ops.dwconv_plan_select(d, pas, -1)
    if layout == NCHW and ops.dwconv_plan(d, 3)["variant_name"] != "none":
        ws = torch.zeros(max(16, ops.dwconv_bwd_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
        ops.dwconv_bwd(d, x, dy, w, dx, dw, ws)
    torch.cuda.synchronize()
    print(f"{name}: ok", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--all-candidates", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--skip-variant", default="", help="comma list of candidate variants not to launch")
    a = ap.parse_args()
    for c in CASES:
        if not a.only or c[0] in a.only.split(","):
            run(*c, a.all_candidates, tuple(v for v in a.skip_variant.split(",") if v))

"""Per-kernel timing the way bench.py measures it (back-to-back launches from a CUDA
graph cycling over copies of the tensors whose footprint is >= 2x L2), for a list
of (layer, pass), plus the same harness around torch's copy_ of the same byte
count (the practical floor for a kernel that reads |in| and writes |out| bytes).

    python tools/kbench.py --layers dw14,dw26 --passes fwd,bwd_filter [--copy]
Planner env knobs (DWCONV_FD_FORCE, DWCONV_BF_FORCE, ...) apply per process, in a library built with
-DDWCONV_DEV_KNOBS only (the shipped build ignores the environment).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1803_09926_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="dw14")
ap.add_argument("--passes", default="fwd,bwd_data,bwd_filter")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--alpha", type=float, default=1.0)
ap.add_argument("--res", type=int, default=224)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--layout", default="nchw")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--copy", action="store_true", help="also time torch copy_ of |in| -> |out| bytes")
ap.add_argument("--tag", default="")
a = ap.parse_args()
dev = torch.device("cuda")
dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
eb = 4 if a.dtype == "f32" else 2
lay = 0 if a.layout == "nchw" else 1
mf = torch.contiguous_format if lay == 0 else torch.channels_last
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
stream = torch.cuda.Stream()


def graph_time(fns):
    """mean µs per call of the callables in `fns`, launched back to back from one graph"""
    with torch.cuda.stream(stream):
        for f in fns:
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(2):
                for f in fns:
                    f()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        for _ in range(a.reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (a.reps * 2 * len(fns))


for lname in a.layers.split(","):
    L = [l for l in synth.mobilenet_v1_dw(a.batch, a.alpha, a.res) if l.name == lname][0]
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, lay, 0 if a.dtype == "f32" else 1)
    xb, yb = L.x_elems() * eb, L.y_elems() * eb
    nsets = int(max(2, min(16, -(-2 * l2 // (2 * (xb + yb))))))
    w = torch.randn(L.c * L.m, L.k, L.k, device=dev).to(dt)
    dw = torch.empty(L.c * L.m, L.k, L.k, device=dev)
    ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device=dev)
    sets = []
    for _ in range(nsets):
        x = torch.randn(L.n, L.c, L.h, L.w, device=dev).to(dt).contiguous(memory_format=mf)
        dy = torch.randn(L.n, L.c * L.m, L.ho, L.wo, device=dev).to(dt).contiguous(memory_format=mf)
        sets.append(dict(x=x, dy=dy, y=torch.empty_like(dy), dx=torch.empty_like(x)))
    for pas in a.passes.split(","):
        mk = {"fwd": lambda s: (lambda: ops.dwconv_fwd(d, s["x"], w, s["y"])),
              "bwd_data": lambda s: (lambda: ops.dwconv_bwd_data(d, s["dy"], w, s["dx"])),
              "bwd_filter": lambda s: (lambda: ops.dwconv_bwd_filter(d, s["x"], s["dy"], dw, ws))}[pas]
        us = graph_time([mk(s) for s in sets])
        nbytes = xb + yb
        pl = ops.dwconv_plan(d, {"fwd": 0, "bwd_data": 1, "bwd_filter": 2}[pas])
        plan = " ".join(f"{k}={pl[k]}" for k in ("grid", "block", "smem_bytes", "planes_per_chunk", "rows_per_band",
                                                  "batch_slices"))
        line = f"{a.tag} {lname} {pas} {us:.2f} us {nbytes / us / 1e3:.0f} GB/s  {plan}"
        if a.copy and pas == "fwd":
            src = [torch.empty(xb // 4, dtype=torch.float32, device=dev) for _ in range(nsets)]
            dst = [torch.empty(yb // 4, dtype=torch.float32, device=dev) for _ in range(nsets)]
            n = min(xb, yb) // 4
            cu = graph_time([(lambda i=i: dst[i][:n].copy_(src[i][:n])) for i in range(nsets)])
            line += f" | copy {2 * n * 4 / 1e6:.1f} MB {cu:.2f} us {2 * n * 4 / cu / 1e3:.0f} GB/s"
        print(line, flush=True)

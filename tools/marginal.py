"""In-context cost of each launch of the 13-layer step: time the CUDA graph of the
whole step (serial order) and the graph with one launch left out; the difference
is that launch's marginal cost with its neighbours overlapping it (PDL) and cold
inputs (step footprint >> L2).  Event-isolated per-kernel timings include a
~5 us launch floor each; this does not.

    python tools/marginal.py [--batch 64] [--dtype f32] [--reps 30] [--only dw14,dw26]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1803_09926_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--only", default="")
ap.add_argument("--fused", action="store_true", help="use dwconv_bwd for layers that have a fused kernel")
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
eb = 4 if a.dtype == "f32" else 2
layers = synth.mobilenet_v1_dw(a.batch)
launches = []
bufs = []
for L in layers:
    d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, 0, 0 if a.dtype == "f32" else 1)
    b = dict(L=L, d=d, x=torch.randn(L.n, L.c, L.h, L.w, device="cuda").to(dt),
             dy=torch.randn(L.n, L.c * L.m, L.ho, L.wo, device="cuda").to(dt),
             w=torch.randn(L.c * L.m, L.k, L.k, device="cuda").to(dt))
    b["y"] = torch.empty_like(b["dy"]); b["dx"] = torch.empty_like(b["x"])
    b["dw"] = torch.empty(L.c * L.m, L.k, L.k, device="cuda")
    b["ws"] = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
    b["wsf"] = torch.zeros(max(16, ops.dwconv_bwd_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
    b["fused"] = a.fused and ops.dwconv_plan(d, 3)["variant_name"] != "none"
    bufs.append(b)
for b in bufs:
    launches.append((b["L"].name, "fwd", (b["x"].numel() + b["y"].numel()) * eb,
                     lambda b=b: ops.dwconv_fwd(b["d"], b["x"], b["w"], b["y"])))
for b in reversed(bufs):
    if b["fused"]:
        launches.append((b["L"].name, "bwd", (2 * b["x"].numel() + b["y"].numel()) * eb,
                         lambda b=b: ops.dwconv_bwd(b["d"], b["x"], b["dy"], b["w"], b["dx"], b["dw"], b["wsf"])))
        continue
    launches.append((b["L"].name, "bwd_data", (b["x"].numel() + b["y"].numel()) * eb,
                     lambda b=b: ops.dwconv_bwd_data(b["d"], b["dy"], b["w"], b["dx"])))
    launches.append((b["L"].name, "bwd_filter", (b["x"].numel() + b["y"].numel()) * eb,
                     lambda b=b: ops.dwconv_bwd_filter(b["d"], b["x"], b["dy"], b["dw"], b["ws"])))

stream = torch.cuda.Stream()


def graph_of(skip):
    with torch.cuda.stream(stream):
        for i, l in enumerate(launches):
            if i != skip:
                l[3]()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i, l in enumerate(launches):
                if i != skip:
                    l[3]()
    torch.cuda.synchronize()
    return g


def time_graph(g):
    with torch.cuda.stream(stream):
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        for _ in range(a.reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.reps


full = time_graph(graph_of(-1))
print(f"full step (serial graph): {full:.1f} us")
only = set(a.only.split(",")) if a.only else None
tot = 0.0
for i, (name, pas, nbytes, _) in enumerate(launches):
    if only and name not in only:
        continue
    t = full - time_graph(graph_of(i))
    tot += t
    print(f"{name:5s} {pas:10s} marginal {t:7.2f} us  {nbytes / max(t, 1e-3) / 1e3:7.0f} GB/s", flush=True)
print(f"sum of marginals {tot:.1f} us")

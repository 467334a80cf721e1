"""Time one (layer, pass) at several batch sizes: separates per-launch fixed cost from per-byte cost."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1803_09926_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="dw2,dw14,dw26")
ap.add_argument("--passes", default="fwd,bwd_data,bwd_filter")
ap.add_argument("--batches", default="16,64,256")
ap.add_argument("--dtype", default="f32")
ap.add_argument("--layout", default="nchw", choices=["nchw", "nhwc"])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--plan", action="store_true", help="append the chosen plan of the last batch")
ap.add_argument("--flush-mb", type=int, default=256, help="bytes read between reps to evict L2 (keeps the GPU busy while the host enqueues)")
ap.add_argument("--graph", action="store_true", help="replay the launch from a CUDA graph (no host launch overhead)")
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
eb = 4 if a.dtype == "f32" else 2
flush = torch.ones(a.flush_mb << 18, dtype=torch.float32, device="cuda")  # 256 MB, read to evict L2 cleanly
sink = torch.empty(1, device="cuda")
for lname in a.layers.split(","):
    for pas in a.passes.split(","):
        row = []
        for n in [int(b) for b in a.batches.split(",")]:
            L = [l for l in synth.mobilenet_v1_dw(n) if l.name == lname][0]
            lay = 0 if a.layout == "nchw" else 1
            mf = torch.contiguous_format if lay == 0 else torch.channels_last
            d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, lay, 0 if a.dtype == "f32" else 1)
            x = torch.randn(L.n, L.c, L.h, L.w, device="cuda").to(dt).contiguous(memory_format=mf)
            dy = torch.randn(L.n, L.c * L.m, L.ho, L.wo, device="cuda").to(dt).contiguous(memory_format=mf)
            w = torch.randn(L.c * L.m, L.k, L.k, device="cuda").to(dt)
            y = torch.empty_like(dy); dx = torch.empty_like(x)  # empty_like keeps the memory format
            dw = torch.empty(L.c * L.m, L.k, L.k, device="cuda")
            ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
            wsf = torch.zeros(max(16, ops.dwconv_bwd_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
            f = {"fwd": lambda: ops.dwconv_fwd(d, x, w, y), "bwd_data": lambda: ops.dwconv_bwd_data(d, dy, w, dx),
                 "bwd_filter": lambda: ops.dwconv_bwd_filter(d, x, dy, dw, ws),
                 "bwd": lambda: ops.dwconv_bwd(d, x, dy, w, dx, dw, wsf)}[pas]
            for _ in range(3): f()
            if a.graph:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    f()
                f = g.replay
            times = []
            for _ in range(a.reps):
                torch.sum(flush, dim=0, keepdim=True, out=sink)
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); f(); e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3)
            times.sort()
            us = times[len(times) // 2]
            nbytes = (L.x_elems() + L.y_elems()) * eb * (2 if pas == "bwd" else 1) - (L.y_elems() * eb if pas == "bwd" else 0)
            row.append((n, round(us, 2), round(nbytes / us / 1e3)))
        extra = ""
        if a.plan:
            pi = ops.dwconv_plan(d, {"fwd": 0, "bwd_data": 1, "bwd_filter": 2, "bwd": 3}[pas])
            extra = " ".join(f"{k}={pi[k]}" for k in ("variant_name", "grid", "block", "smem_bytes", "planes_per_chunk",
                                                      "rows_per_band", "batch_slices"))
        print(lname, pas, row, extra, flush=True)

"""Time every candidate plan of a pass on arbitrary shapes (bench.py's per-kernel harness: back-to-back
launches from a CUDA graph over rotating tensor copies >= 2x L2, CUDA events on the launching stream).

Used for the block-diagonal tensor-core sweep (the B200 analogue of PAPER.md Fig. 5,
P:600-622: time vs group size S) and the configs[3] stress shapes.

    python tools/sweep_candidates.py --shapes cfg4 --dtype bf16 --layout nhwc --passes fwd,bwd_data --json out.json

Each row: shape, pass, candidate (variant, S for the tensor-core variant), mean µs, algorithmic GB/s and
fraction of the measured copy peak, useful FMA/s (N*C*m*Ho*Wo*K^2 / t) and, for the tensor-core variant,
the MMA rate the hardware executed (useful x S).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1803_09926_b200 import ops  # noqa: E402
from paper_1803_09926_b200._lib import BF16, F32, NCHW, NHWC  # noqa: E402

SETS = {
    # configs[3], batch 64
    "cfg4": [(64, 128, 56, 56, 2, 3, 1, 1), (64, 128, 56, 56, 4, 3, 1, 1), (64, 128, 56, 56, 1, 5, 1, 2),
             (64, 128, 56, 56, 1, 7, 1, 3), (64, 512, 56, 56, 1, 3, 2, 1), (64, 512, 56, 56, 1, 5, 2, 2),
             (64, 512, 56, 56, 1, 7, 2, 3)],
    # MobileNet-v1 layers at batch 128 (the >= 70 % target set): large planes and the 14x14 / 7x7 layers
    "mb128": [(128, 32, 112, 112, 1, 3, 1, 1), (128, 64, 112, 112, 1, 3, 2, 1), (128, 128, 56, 56, 1, 3, 1, 1),
              (128, 512, 14, 14, 1, 3, 1, 1), (128, 512, 14, 14, 1, 3, 2, 1), (128, 1024, 7, 7, 1, 3, 1, 1)],
    # the same layers at batch 64 (configs[1], the fp32 headline)
    "mb64": [(64, 32, 112, 112, 1, 3, 1, 1), (64, 64, 112, 112, 1, 3, 2, 1), (64, 128, 56, 56, 1, 3, 1, 1),
             (64, 512, 14, 14, 1, 3, 1, 1), (64, 512, 14, 14, 1, 3, 2, 1), (64, 1024, 7, 7, 1, 3, 1, 1)],
    # the group-size sweep: stride-1 K = 3 / 5 / 7 on 56x56x128 (b64) and a MobileNet 3x3 layer (dw6, b128)
    "sweep": [(64, 128, 56, 56, 1, 3, 1, 1), (64, 128, 56, 56, 1, 5, 1, 2), (64, 128, 56, 56, 1, 7, 1, 3),
              (128, 128, 56, 56, 1, 3, 1, 1), (128, 512, 14, 14, 1, 3, 1, 1)],
}
PASSES = {"fwd": 0, "bwd_data": 1, "bwd_filter": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="sweep")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--layout", default="nhwc")
    ap.add_argument("--passes", default="fwd,bwd_data")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = float(peaks["hbm_gbs"])
    dev = torch.device("cuda")
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    eb = 4 if a.dtype == "f32" else 2
    lay = NCHW if a.layout == "nchw" else NHWC
    mf = torch.channels_last if lay == NHWC else torch.contiguous_format
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    stream = torch.cuda.Stream()
    rows = []
    for shp in SETS[a.shapes]:
        N, C, H, W, m, K, s, p = shp
        d = ops.make_desc(N, C, H, W, m, K, s, p, lay, F32 if a.dtype == "f32" else BF16)
        Ho, Wo = ops.output_shape(d)
        x = torch.randn(N, C, H, W, device=dev).to(tdt).contiguous(memory_format=mf)
        dy = torch.randn(N, C * m, Ho, Wo, device=dev).to(tdt).contiguous(memory_format=mf)
        w = torch.randn(C * m, K, K, device=dev).to(tdt)
        set_bytes = (x.numel() + dy.numel()) * eb * 2
        nsets = int(max(2, min(8, -(-2 * l2 // set_bytes))))
        sets = [dict(x=x if i == 0 else x.clone(), dy=dy if i == 0 else dy.clone(), y=torch.empty_like(dy),
                     dx=torch.empty_like(x)) for i in range(nsets)]
        dw = torch.empty(C * m, K, K, device=dev)
        fma = N * C * m * Ho * Wo * K * K
        for pname in a.passes.split(","):
            pas = PASSES[pname]
            cands = ops.dwconv_plan_candidates(d, pas) or [None]
            ws = torch.zeros(max([16, ops.dwconv_bwd_filter_workspace_bytes(d)] +
                                 [c["workspace_bytes"] for c in cands if c]), dtype=torch.uint8, device=dev)

            def mk(st):
                if pas == 0:
                    return lambda: ops.dwconv_fwd(d, st["x"], w, st["y"])
                if pas == 1:
                    return lambda: ops.dwconv_bwd_data(d, st["dy"], w, st["dx"])
                return lambda: ops.dwconv_bwd_filter(d, st["x"], st["dy"], dw, ws)

            for i, c in enumerate(cands):
                if c is not None:
                    ops.dwconv_plan_select(d, pas, i)
                fns = [mk(st) for st in sets] * 2
                stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(stream):
                    for f in fns:
                        f()
                    torch.cuda.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
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
                us = e0.elapsed_time(e1) * 1e3 / (a.reps * len(fns))
                del g
                nbytes = (x.numel() + dy.numel() + w.numel()) * eb + (dw.numel() * 4 if pas == 2 else 0)
                var = c["variant_name"] if c else ops.dwconv_plan(d, pas)["variant_name"]
                S = c["planes_per_chunk"] if (c and var == "nhwc_bdmma") else None
                CB = c["rows_per_band"] if (c and var == "nhwc_bdmma") else None
                r = dict(shape=dict(N=N, C=C, H=H, W=W, m=m, K=K, s=s, p=p), dtype=a.dtype, layout=a.layout,
                         pass_=pname, candidate=i, variant=var, S=S, CB=CB, us=us, gbs=nbytes / us / 1e3,
                         frac=nbytes / us / 1e3 / peak, useful_tfma=fma / us / 1e6,
                         mma_tflops=(2 * fma * S / us / 1e6) if S else None,
                         grid=c["grid"] if c else None, block=c["block"] if c else None,
                         family=c["kernel_family"] if c else None, slices=c["batch_slices"] if c else None)
                rows.append(r)
                print(json.dumps(r), flush=True)
            if cands[0] is not None:
                ops.dwconv_plan_select(d, pas, -1)
        del sets, x, dy
        torch.cuda.empty_cache()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: MobileNet-v1 depthwise fwd+bwd images/s and achieved HBM GB/s on B200.

A step is one pass of the whole hot path over one batch: the 13 depthwise 3x3
layers of MobileNet-v1 (Table III) forward, then
bwd_data + bwd_filter in reverse layer order (39 kernels of libdwconv.so),
plus, at N > 1 GPUs, one NCCL all_reduce(SUM) of the flat filter-gradient
bucket (44,640 fp32).  Default workload: BASELINE.json configs[1] -- width 1.0,
224 px, batch 64 per GPU, fp32, NCHW.  Inputs are seeded synthetic U[-1,1].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MobileNet-v1 depthwise fwd+bwd images/s and achieved HBM GB/s (% peak), 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
PAPER_CONTEXT_IMG_S = 445.0  # Table III Diagonalwise cuDNN fwd+bwd, x5-corrected, GTX 1080 Ti


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="images per GPU")
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--layout", default="nchw", choices=["nchw", "nhwc"])
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying a CUDA graph")
    ap.add_argument("--serial", action="store_true", help="all 39 launches on one stream (no dgrad/wgrad overlap)")
    ap.add_argument("--fused", default="none", choices=["none", "all", "small"],
                    help="layers whose backward uses the fused dwconv_bwd (one pass over x and dy) instead of "
                         "bwd_data + bwd_filter on two streams: none, all fusable, or the fusable 14x14/7x7 layers")
    ap.add_argument("--no-tune", action="store_true", help="keep the planner's launch shapes (no measured selection)")
    ap.add_argument("--plans", default="", help="JSON file of measured plan selections: loaded if it exists, else written")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget (cpu_baseline)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--kernel-reps", type=int, default=5, help="graph replays per kernel in the per-kernel timing")
    ap.add_argument("--extra", action="store_true", help="add per-layer kernel table to the JSON line")
    return ap.parse_args()


def layers_for(args, batch):
    import synth
    return synth.mobilenet_v1_dw(batch, alpha=args.alpha, resolution=args.res)


def workload_name(args):
    w = f"mobilenet_v1_a{args.alpha:g}_r{args.res}_dw13"
    return w


def step_bytes(layers, eb, fused=None):
    """Algorithmic HBM bytes of one fwd+bwd step: 3|x| + 3|y| + 2|w| + |dw| per
    layer; a layer whose backward is fused (dwconv_bwd, NEXT-1) reads dy once: 3|x| + 2|y| + ..."""
    tot = 0
    for i, L in enumerate(layers):
        ny = 2 if (fused and fused[i]) else 3
        tot += 3 * L.x_elems() * eb + ny * L.y_elems() * eb + 2 * L.w_elems() * eb + L.w_elems() * 4
    return tot


def pass_bytes(L, pas, eb):
    if pas == "fwd":
        return (L.x_elems() + L.y_elems() + L.w_elems()) * eb
    if pas == "bwd_data":
        return (L.x_elems() + L.y_elems() + L.w_elems()) * eb
    if pas == "bwd":  # fused: x, dy, w read; dx, dw written
        return (2 * L.x_elems() + L.y_elems() + L.w_elems()) * eb + L.w_elems() * 4
    return (L.x_elems() + L.y_elems()) * eb + L.w_elems() * 4


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML while the timed region runs."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for bit, name in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ oracle timing (CPU)
def oracle_sample(layers, s_budget, max_images=64):
    """Time the oracle on images of the workload until ~s_budget seconds; returns (img/s, images, secs)."""
    import oracle
    import synth
    oracle.build()
    t0 = time.perf_counter()
    done = 0
    while done < max_images:
        for li, L in enumerate(layers):
            x = synth.uniform(synth.layer_seed(li, "x"), (1, L.c, L.h, L.w), start=done * L.c * L.h * L.w)
            w = synth.uniform(synth.layer_seed(li, "w"), (L.c * L.m, L.k, L.k))
            dy = synth.uniform(synth.layer_seed(li, "dy"), (1, L.c * L.m, L.ho, L.wo),
                               start=done * L.c * L.m * L.ho * L.wo)
            oracle.fwd(x, w, L.s, L.p)
            oracle.bwd_data(dy, w, x.shape, L.s, L.p)
            oracle.bwd_filter(x, dy, w.shape, L.s, L.p)
        done += 1
        if time.perf_counter() - t0 >= s_budget:
            break
    secs = time.perf_counter() - t0
    return done / secs, done, secs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    layers = layers_for(args, 1)
    import oracle
    oracle.build()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle_sample(layers, 0.0, max_images=1)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = 1000.0 / ms
    eb = 4 if args.dtype == "f32" else 2
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 U[-1,1])",
        "config": {"workload": workload_name(args), "batch_per_gpu": args.batch, "dtype_storage": args.dtype,
                   "layout": args.layout, "sample": "1 image per step"},
        "hbm_gbs": None,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": 1, "kind": "oracle",
                         "sample": "each step = 1 image of the 13-layer stack, fwd+bwd_data+bwd_filter, "
                                   "plain-C fp64 oracle, single thread"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "algorithmic_bytes_per_image": step_bytes(layers, eb),
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_1803_09926_b200 as dwl
    from paper_1803_09926_b200 import dp, ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    layout = dwl.NCHW if args.layout == "nchw" else dwl.NHWC
    dcode = dwl.F32 if args.dtype == "f32" else dwl.BF16
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    eb = 4 if args.dtype == "f32" else 2
    mf = torch.channels_last if layout == dwl.NHWC else torch.contiguous_format
    layers = layers_for(args, args.batch)

    # ---- buffers: distinct per layer; weights and dw bucket shared (flat)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def rnd(shape, dtype=tdt):
        t = torch.empty(shape, dtype=torch.float32, device=dev).uniform_(-1.0, 1.0, generator=gen)
        return t.to(dtype).contiguous(memory_format=mf) if len(shape) == 4 else t.to(dtype)

    bucket = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in layers], device=dev)  # every layer's dw, one all-reduce
    dw_bucket = bucket.flat
    bufs = []
    for L in layers:
        d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, layout, dcode)
        b = dict(L=L, d=d, x=rnd((L.n, L.c, L.h, L.w)), w=rnd((L.c * L.m, L.k, L.k)),
                 dy=rnd((L.n, L.c * L.m, L.ho, L.wo)),
                 y=torch.empty((L.n, L.c * L.m, L.ho, L.wo), dtype=tdt, device=dev, memory_format=mf),
                 dx=torch.empty((L.n, L.c, L.h, L.w), dtype=tdt, device=dev, memory_format=mf),
                 dw=bucket.views[len(bufs)],
                 wsb=ops.dwconv_bwd_filter_workspace_bytes(d))
        bufs.append(b)
    # fused backward (dx + dw in one pass over x and dy) where the library has the kernel
    for b in bufs:
        b["fused"] = (args.fused == "all" or (args.fused == "small" and b["L"].h <= 14)) and \
            ops.dwconv_plan(b["d"], 3)["variant_name"] != "none"
    # measured plan selection (tune.py): time every candidate launch shape of each
    # pass on this layer's tensors and keep the fastest (before any graph capture)
    tuned = {}
    if not args.no_tune:
        from paper_1803_09926_b200 import tune
        saved = None
        if args.plans and os.path.exists(args.plans):
            with open(args.plans) as f:
                saved = json.load(f)
        for b in bufs:
            if saved is not None:  # re-install a saved selection (no timing: e.g. under ncu)
                tuned[b["L"].name] = saved[b["L"].name]
                tune.apply_selection(b["d"], tuned[b["L"].name])
            else:
                tuned[b["L"].name] = tune.tune_layer(b["d"], b["x"], b["dy"], b["w"],
                                                     passes=("fwd", "bwd") if b["fused"] else
                                                     ("fwd", "bwd_data", "bwd_filter"))
            b["wsb"] = ops.dwconv_bwd_filter_workspace_bytes(b["d"])
        torch.cuda.synchronize()
        if args.plans and saved is None and rank == 0:
            with open(args.plans, "w") as f:
                json.dump(tuned, f)
    ws = torch.zeros(max(16, max(b["wsb"] for b in bufs)), dtype=torch.uint8, device=dev)
    footprint = sum(b[k].numel() * b[k].element_size() for b in bufs for k in ("x", "w", "dy", "y", "dx"))

    def launch_fwd(b):
        ops.dwconv_fwd(b["d"], b["x"], b["w"], b["y"])

    def launch_bd(b):
        ops.dwconv_bwd_data(b["d"], b["dy"], b["w"], b["dx"])

    def launch_bf(b):
        ops.dwconv_bwd_filter(b["d"], b["x"], b["dy"], b["dw"], ws)

    wsf = torch.zeros(max([16] + [ops.dwconv_bwd_workspace_bytes(b["d"]) for b in bufs if b["fused"]]),
                      dtype=torch.uint8, device=dev)

    def launch_bwd(b):
        ops.dwconv_bwd(b["d"], b["x"], b["dy"], b["w"], b["dx"], b["dw"], wsf)

    kernels = [("fwd", b, launch_fwd) for b in bufs]
    for b in reversed(bufs):
        kernels += [("bwd", b, launch_bwd)] if b["fused"] else [("bwd_data", b, launch_bd), ("bwd_filter", b, launch_bf)]

    side = torch.cuda.Stream(device=dev)

    def step_kernels():
        """fwd 13 layers, then per layer (reverse order) bwd_data on the main stream and
        bwd_filter on a side stream.  bwd_filter(L) needs only x_L and dy_L, so it may
        run as soon as dy_L exists (here: when the main stream reaches layer L's
        backward) and overlaps the remaining input-gradient chain -- the dependency
        structure of a real training step (dw is off the critical path).  --serial
        keeps every launch on one stream."""
        if args.serial:
            for _, b, f in kernels:
                f(b)
            return
        cur = torch.cuda.current_stream()
        for b in bufs:
            launch_fwd(b)
        for b in reversed(bufs):
            if b["fused"]:
                launch_bwd(b)
                continue
            ev = torch.cuda.Event()
            ev.record(cur)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                launch_bf(b)
            launch_bd(b)
        ev = torch.cuda.Event()
        ev.record(side)
        cur.wait_event(ev)

    stream = torch.cuda.Stream(device=dev)
    graph = None
    with torch.cuda.stream(stream):
        for _ in range(3):
            step_kernels()
        torch.cuda.synchronize()
        if not args.no_graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step_kernels()
            torch.cuda.synchronize()

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            step_kernels()
        if world > 1:
            bucket.allreduce()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides, CUDA events on the launching stream
    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
    torch.cuda.synchronize()
    sampler.stop()
    if world > 1:
        dist.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    images = args.batch * world
    value = images / (ms / 1000.0)
    sbytes = step_bytes(layers, eb, [b["fused"] for b in bufs])
    hbm_gbs = sbytes * world / (ms / 1000.0) / 1e9

    # ---- per-kernel durations: back-to-back launches of one kernel from a CUDA graph,
    # cycling over enough copies of its tensors that their footprint is >= 2x L2 (inputs
    # come from HBM), CUDA events around the replay on the launching stream
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    reps = args.kernel_reps  # 0: skip (e.g. under ncu, so the last launches are one step in order)
    kt = []
    for pas, b, f in (kernels if reps > 0 else []):
        L = b["L"]
        set_bytes = sum(b[k].numel() * b[k].element_size() for k in ("x", "dy", "y", "dx"))
        nsets = int(max(2, min(16, -(-2 * l2 // set_bytes))))
        sets = [b] + [dict(b, x=torch.empty_like(b["x"]), dy=torch.empty_like(b["dy"]), y=torch.empty_like(b["y"]),
                           dx=torch.empty_like(b["dx"])) for _ in range(nsets - 1)]
        for bs in sets[1:]:
            bs["x"].copy_(b["x"]); bs["dy"].copy_(b["dy"])
        nl = 2 * nsets
        with torch.cuda.stream(stream):
            for bs in sets:
                f(bs)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for j in range(nl):
                    f(sets[j % nsets])
            g.replay()
            torch.cuda.synchronize()
            e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_a.record(stream)
            for _ in range(reps):
                g.replay()
            e_b.record(stream)
        torch.cuda.synchronize()
        mean_ms = e_a.elapsed_time(e_b) / (reps * nl)
        del g, sets
        nbytes = pass_bytes(L, pas, eb)
        kt.append(dict(layer=L.name, pass_=pas, ms=mean_ms, bytes=nbytes, gbs=nbytes / (mean_ms * 1e-3) / 1e9))
        if args.extra:
            pl = ops.dwconv_plan(b["d"], {"fwd": 0, "bwd_data": 1, "bwd_filter": 2, "bwd": 3}[pas])
            kt[-1]["plan"] = {k: pl[k] for k in ("variant_name", "grid", "block", "smem_bytes", "work_units",
                                                 "planes_per_chunk", "rows_per_band", "batch_slices")}
    kernel_sum_ms = sum(k["ms"] for k in kt)
    dom = max(kt, key=lambda k: k["ms"]) if kt else dict(layer="-", pass_="-", ms=float("nan"), bytes=0,
                                                         gbs=float("nan"))
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            peak = float(json.load(f)["hbm_gbs"])
        peak_src = "measured"
    else:
        peak, peak_src = FALLBACK_HBM_GBS, "fallback"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f)
            key = f"{args.alpha:g}/{args.res}/{args.batch}/{args.dtype}/{args.layout}/{dom['layer']}/{dom['pass_']}"
            traffic = tr.get(key)
        except Exception:
            traffic = None
    passes = {}
    for pas in ("fwd", "bwd_data", "bwd_filter", "bwd"):
        sel = [k for k in kt if k["pass_"] == pas]
        if not sel:
            continue
        pm = sum(k["ms"] for k in sel)
        pb = sum(k["bytes"] for k in sel)
        passes[pas] = {"ms": pm, "gbs": pb / (pm * 1e-3) / 1e9, "frac": pb / (pm * 1e-3) / 1e9 / peak}

    # ---- end to end through the public binding with host buffers (pinned), eager calls
    e2e = None
    if args.e2e_steps > 0:
        host_in = []
        for b in bufs:
            host_in.append((b["x"].cpu().pin_memory(), b["dy"].cpu().pin_memory(), b["w"].cpu().pin_memory()))
        host_dw = torch.empty(dw_bucket.shape, dtype=torch.float32).pin_memory()
        h2d = sum(t.numel() * t.element_size() for tup in host_in for t in tup)
        d2h = host_dw.numel() * 4

        def e2e_step():
            for b, (hx, hdy, hw) in zip(bufs, host_in):
                b["x"].copy_(hx, non_blocking=True)
                b["dy"].copy_(hdy, non_blocking=True)
                b["w"].copy_(hw, non_blocking=True)
            step_kernels()
            if world > 1:
                bucket.allreduce()
            host_dw.copy_(dw_bucket, non_blocking=True)

        with torch.cuda.stream(stream):
            e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(args.e2e_steps):
                e2e_step()
            f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": images / (e2e_ms / 1000.0), "unit": "images/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "path": "python binding -> C ABI eager calls; pinned host->device copies of x, dy, w for all "
                       "13 layers and device->host copy of the dw bucket inside the timed region"}

    # ---- CPU baseline (oracle), rank 0 at N=1 only
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        v, nimg, secs = oracle_sample(layers_for(args, 1), args.cpu_seconds)
        cpu = {"value": v, "unit": "images/s", "cores": 1, "kind": "oracle",
               "sample": f"{nimg} images of the 13-layer stack (fwd+bwd_data+bwd_filter), plain-C fp64 oracle, "
                         f"single thread, {secs:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded torch U[-1,1] on device; parity tests use the splitmix64 generator)",
            "config": {"workload": workload_name(args), "global_batch": images, "batch_per_gpu": args.batch,
                       "layers": 13, "layout": args.layout, "parallelism": f"dp{world}",
                       "l2": f"no flush: step footprint {footprint / 1e9:.2f} GB >> 126 MB L2",
                       "graph": graph is not None,
                       "schedule": ("serial" if args.serial else "bwd_filter on a side stream (overlaps bwd_data)") +
                                   f"; fused backward on {sum(b['fused'] for b in bufs)}/13 layers",
                       "plans": ("planner defaults" if not tuned else
                                 "measured selection (tune.py, before the timed region): "
                                 f"{sum(1 for t in tuned.values() for v in t.values() if v['index'] != 0)} of "
                                 f"{sum(len(t) for t in tuned.values())} tuned passes changed")},
            "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / world / peak,
            "algorithmic_bytes_per_step": sbytes * world,
            "roofline": ({"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                          "frac": dom["gbs"] / peak, "traffic": traffic, "peak_source": peak_src,
                          "kernel": f"{dom['layer']}/{dom['pass_']}", "ms": dom["ms"], "bytes": dom["bytes"],
                          "timing": "back-to-back graph launches over rotating copies >= 2x L2"} if kt else None),
            "passes": passes,
            "kernel_sum_ms": kernel_sum_ms,
            "clocks": sampler.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": len(kernels) * args.steps,
            "paper_context": {"img_s": PAPER_CONTEXT_IMG_S, "hw": "GTX 1080 Ti, Caffe, Table III (context only)"},
        }
        if args.extra:
            line["tuning"] = tuned
            line["kernels"] = [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in kk.items()} for kk in kt]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

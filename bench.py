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
    torchrun --nproc-per-node N bench.py --gpus N --global-batch 1024   # configs[4], strong scaling

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every field).  At N=1 the
line also carries ``workloads_b128``: the north star's >= 70 % target set
(alpha 1.0 / 224 at batch 128: fp32 NCHW, bf16 NCHW, bf16 NHWC), each measured
the same way in the same process.
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
NOMINAL_HBM_GBS = 8000.0          # BASELINE north star "~8 TB/s peak"; the >= 70 % target is stated on it
NVLINK_GBS_PER_DIR = 900.0        # NVLink 5, per GPU per direction (the all-reduce roofline basis)
PAPER_CONTEXT_IMG_S = 445.0  # Table III Diagonalwise cuDNN fwd+bwd, x5-corrected, GTX 1080 Ti
B128_SET = (("f32", "nchw"), ("bf16", "nchw"), ("bf16", "nhwc"))


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64, help="images per GPU (weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="total images split over the ranks with dp.shard_batch (configs[4]: 1024; strong scaling)")
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
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="oracle sample budget per cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--kernel-reps", type=int, default=5, help="graph replays per kernel in the per-kernel timing")
    ap.add_argument("--no-b128", action="store_true", help="skip the batch-128 target-set workloads (N=1 only)")
    ap.add_argument("--b128-steps", type=int, default=50)
    ap.add_argument("--extra", action="store_true", help="add per-layer kernel table to the JSON line")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend at N > 1 (gloo + --one-device: exercise the N > 1 path on one GPU)")
    ap.add_argument("--one-device", action="store_true", help="put every rank on cuda:0 (test mode)")
    return ap.parse_args(argv)


def layers_for(alpha, res, batch):
    import synth
    return synth.mobilenet_v1_dw(batch, alpha=alpha, resolution=res)


def workload_name(alpha, res):
    return f"mobilenet_v1_a{alpha:g}_r{res}_dw13"


def step_bytes(layers, eb, fused=None):
    """Algorithmic HBM bytes of one fwd+bwd step: 3|x| + 3|y| + 2|w| + |dw| per
    layer; a layer whose backward is fused (dwconv_bwd, NEXT-1) reads dy once: 3|x| + 2|y| + ..."""
    tot = 0
    for i, L in enumerate(layers):
        ny = 2 if (fused and fused[i]) else 3
        tot += 3 * L.x_elems() * eb + ny * L.y_elems() * eb + 2 * L.w_elems() * eb + L.w_elems() * 4
    return tot


def pass_bytes(L, pas, eb):
    if pas in ("fwd", "bwd_data"):
        return (L.x_elems() + L.y_elems() + L.w_elems()) * eb
    if pas == "bwd":  # fused: x, dy, w read; dx, dw written
        return (2 * L.x_elems() + L.y_elems() + L.w_elems()) * eb + L.w_elems() * 4
    return (L.x_elems() + L.y_elems()) * eb + L.w_elems() * 4


def dev_env():
    """DWCONV_* variables in the environment.  The shipped library reads none of them (launch-shape knobs
    exist only in a -DDWCONV_DEV_KNOBS build), so they cannot change a timed launch; recorded anyway."""
    return {k: v for k, v in os.environ.items() if k.startswith("DWCONV_")}


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
def oracle_sample(layers, s_budget, max_images=64, threads=1):
    """Time the oracle on images of the workload until ~s_budget seconds; returns (img/s, images, secs)."""
    import oracle
    import synth
    oracle.build()
    oracle.set_threads(threads)
    try:
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
    finally:
        oracle.set_threads(1)
    return done / secs, done, secs


def oracle_threads_bitwise(layers, threads):
    """The all-cores oracle must give bitwise the single-thread results: checked on one
    image of the last layer (all three passes) before its time is reported."""
    import oracle
    import synth
    li = len(layers) - 1
    L = layers[li]
    x = synth.uniform(synth.layer_seed(li, "x"), (2, L.c, L.h, L.w))
    w = synth.uniform(synth.layer_seed(li, "w"), (L.c * L.m, L.k, L.k))
    dy = synth.uniform(synth.layer_seed(li, "dy"), (2, L.c * L.m, L.ho, L.wo))
    outs = []
    for t in (1, threads):
        oracle.set_threads(t)
        outs.append([oracle.fwd(x, w, L.s, L.p), oracle.bwd_data(dy, w, x.shape, L.s, L.p),
                     oracle.bwd_filter(x, dy, w.shape, L.s, L.p)])
    oracle.set_threads(1)
    return all(np.array_equal(a, b) for r1, r2 in zip(*outs) for a, b in zip(r1, r2))


def cpu_baselines(layers, s_budget):
    cores = len(os.sched_getaffinity(0))
    v1, n1, s1 = oracle_sample(layers, s_budget, threads=1)
    single = {"value": v1, "unit": "images/s", "cores": 1, "kind": "oracle",
              "sample": f"{n1} images of the 13-layer stack (fwd+bwd_data+bwd_filter), plain-C fp64 oracle, "
                        f"single thread, {s1:.1f} s"}
    allc = None
    if cores > 1:
        same = oracle_threads_bitwise(layers, cores)
        va, na, sa = oracle_sample(layers, s_budget, max_images=256, threads=cores)
        allc = {"value": va, "unit": "images/s", "cores": cores, "kind": "oracle",
                "bitwise_equal_to_single_thread": same,
                "sample": f"{na} images of the 13-layer stack, same oracle with its outer loops over {cores} "
                          f"OpenMP threads, {sa:.1f} s"}
    return single, allc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    layers = layers_for(args.alpha, args.res, 1)
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
        "config": {"workload": workload_name(args.alpha, args.res), "batch_per_gpu": args.batch,
                   "dtype_storage": args.dtype, "layout": args.layout, "sample": "1 image per step"},
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
def hbm_peak():
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def pct(v, q):
    return float(np.percentile(np.asarray(v, dtype=np.float64), q))


class Workload:
    """Every buffer of one bench workload: NSETS complete input/output sets (x, dy, y, dx per layer) that
    successive steps alternate between, shared weights and one flat dw bucket; the measured plan
    selection; one CUDA graph per set."""
    NSETS = 2

    def __init__(self, torch, dev, rank, alpha, res, batch, dtype, layout, fused_mode="none", tune=True,
                 plans_file="", serial=False, graph=True):
        import paper_1803_09926_b200 as dwl
        from paper_1803_09926_b200 import dp, ops
        self.torch, self.ops, self.dev = torch, ops, dev
        self.alpha, self.res, self.batch, self.dtype, self.layout = alpha, res, batch, dtype, layout
        self.serial = serial
        lay = dwl.NCHW if layout == "nchw" else dwl.NHWC
        dcode = dwl.F32 if dtype == "f32" else dwl.BF16
        tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        self.eb = 4 if dtype == "f32" else 2
        mf = torch.channels_last if lay == dwl.NHWC else torch.contiguous_format
        self.layers = layers_for(alpha, res, batch)
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)

        def rnd(shape):
            t = torch.empty(shape, dtype=torch.float32, device=dev).uniform_(-1.0, 1.0, generator=gen)
            return t.to(tdt).contiguous(memory_format=mf) if len(shape) == 4 else t.to(tdt)

        self.bucket = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in self.layers], device=dev)
        self.descs, self.w, self.fused = [], [], []
        self.sets = [[] for _ in range(self.NSETS)]
        for li, L in enumerate(self.layers):
            d = ops.make_desc(L.n, L.c, L.h, L.w, L.m, L.k, L.s, L.p, lay, dcode)
            self.descs.append(d)
            self.w.append(rnd((L.c * L.m, L.k, L.k)))
            for s in self.sets:
                s.append(dict(x=rnd((L.n, L.c, L.h, L.w)), dy=rnd((L.n, L.c * L.m, L.ho, L.wo)),
                              y=torch.empty((L.n, L.c * L.m, L.ho, L.wo), dtype=tdt, device=dev, memory_format=mf),
                              dx=torch.empty((L.n, L.c, L.h, L.w), dtype=tdt, device=dev, memory_format=mf)))
            self.fused.append((fused_mode == "all" or (fused_mode == "small" and L.h <= 14)) and L.n > 0 and
                              ops.dwconv_plan(d, 3)["variant_name"] != "none")
        # measured plan selection (tune.py): every candidate launch shape of each pass timed on this
        # layer's tensors, the fastest kept as an immutable plan handle (dwconv_plan_create) that every
        # launch below goes through -- no process-wide plan state is installed or read
        self.tuned = {}
        self.plans = []
        from paper_1803_09926_b200 import tune as tn
        saved = None
        if tune and plans_file and os.path.exists(plans_file):
            with open(plans_file) as f:
                saved = json.load(f)
        for li, L in enumerate(self.layers):
            passes = ("fwd", "bwd") if self.fused[li] else ("fwd", "bwd_data", "bwd_filter")
            if tune and L.n > 0 and saved is not None:  # a saved selection (no timing: e.g. under ncu)
                self.tuned[L.name] = saved[L.name]
                self.plans.append(tn.plans_from_selection(self.descs[li], saved[L.name]))
            elif tune and L.n > 0:
                s0 = self.sets[0][li]
                res = tn.tune_layer(self.descs[li], s0["x"], s0["dy"], self.w[li], passes=passes)
                self.plans.append({k: v["plan"] for k, v in res.items()})
                self.tuned[L.name] = tn.selection_json(res)
            else:
                self.plans.append({k: ops.Plan(self.descs[li], tn.PASSES[k], -1) for k in passes})
        torch.cuda.synchronize()
        if tune and plans_file and saved is None and rank == 0:
            with open(plans_file, "w") as f:
                json.dump(self.tuned, f)
        self.ws = torch.zeros(max([16] + [pl["bwd_filter"].workspace_bytes for pl in self.plans if "bwd_filter" in pl]),
                              dtype=torch.uint8, device=dev)
        self.wsf = torch.zeros(max([16] + [pl["bwd"].workspace_bytes for pl in self.plans if "bwd" in pl]),
                               dtype=torch.uint8, device=dev)
        self.footprint = sum(t.numel() * t.element_size() for s in self.sets for b in s for t in b.values())
        self.side = torch.cuda.Stream(device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.graphs = None
        if graph:
            with torch.cuda.stream(self.stream):
                for k in range(self.NSETS):
                    for _ in range(2):
                        self.step_kernels(k)
                torch.cuda.synchronize()
                self.graphs = []
                for k in range(self.NSETS):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.stream):
                        self.step_kernels(k)
                    self.graphs.append(g)
                torch.cuda.synchronize()

    # -- launches (each one call of the C ABI through the binding, on the layer's plan handle)
    def launch(self, pas, li, b):
        pl = self.plans[li][pas]
        if pas == "fwd":
            pl.fwd(b["x"], self.w[li], b["y"])
        elif pas == "bwd_data":
            pl.bwd_data(b["dy"], self.w[li], b["dx"])
        elif pas == "bwd_filter":
            pl.bwd_filter(b["x"], b["dy"], self.bucket.views[li], self.ws)
        else:
            pl.bwd(b["x"], b["dy"], self.w[li], b["dx"], self.bucket.views[li], self.wsf)

    def kernel_list(self):
        ks = [("fwd", li) for li in range(len(self.layers))]
        for li in reversed(range(len(self.layers))):
            ks += [("bwd", li)] if self.fused[li] else [("bwd_data", li), ("bwd_filter", li)]
        return [(p, li) for p, li in ks if self.layers[li].n > 0]

    def step_kernels(self, k):
        """fwd 13 layers, then per layer (reverse order) bwd_data on the main stream and bwd_filter on a
        side stream.  bwd_filter(L) needs only x_L and dy_L, so it may run as soon as dy_L exists (here:
        when the main stream reaches layer L's backward) and overlaps the remaining input-gradient chain
        -- the dependency structure of a real training step (dw is off the critical path).  --serial keeps
        every launch on one stream."""
        torch = self.torch
        s = self.sets[k]
        if self.serial:
            for pas, li in self.kernel_list():
                self.launch(pas, li, s[li])
            return
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        for pas, li in self.kernel_list():
            if pas == "fwd" or pas == "bwd":
                self.launch(pas, li, s[li])
            elif pas == "bwd_data":
                ev = torch.cuda.Event()
                ev.record(cur)
                self.side.wait_event(ev)
                with torch.cuda.stream(self.side):
                    self.launch("bwd_filter", li, s[li])
                self.launch("bwd_data", li, s[li])
        ev = torch.cuda.Event()
        ev.record(self.side)
        cur.wait_event(ev)

    def one_step(self, k):
        if self.graphs is not None:
            self.graphs[k % self.NSETS].replay()
        else:
            self.step_kernels(k % self.NSETS)

    def timed_steps(self, steps, warmup, allreduce=None, barrier=None):
        """K steps alternating the input sets; an event between steps gives the per-step times."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            for i in range(warmup):
                self.one_step(i)
                if allreduce:
                    allreduce()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(self.stream):
            evs[0].record(self.stream)
            for i in range(steps):
                self.one_step(i)
                if allreduce:
                    allreduce()
                evs[i + 1].record(self.stream)
        torch.cuda.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
        return evs[0].elapsed_time(evs[-1]) / steps, per

    def kernel_times(self, reps):
        """Per-kernel durations: back-to-back launches of one kernel from a CUDA graph, cycling over enough
        copies of its tensors that their footprint is >= 2x L2 (inputs come from HBM),
        CUDA events around the replay on the launching stream."""
        torch = self.torch
        l2 = torch.cuda.get_device_properties(self.dev).L2_cache_size
        kt = []
        for pas, li in self.kernel_list():
            L = self.layers[li]
            b = self.sets[0][li]
            set_bytes = sum(b[k].numel() * b[k].element_size() for k in ("x", "dy", "y", "dx"))
            nsets = int(max(2, min(16, -(-2 * l2 // set_bytes))))
            sets = [b, self.sets[1][li]] + [{k: torch.empty_like(v) for k, v in b.items()}
                                            for _ in range(max(0, nsets - 2))]
            for bs in sets[2:]:
                bs["x"].copy_(b["x"])
                bs["dy"].copy_(b["dy"])
            nsets = len(sets)
            nl = 2 * nsets
            with torch.cuda.stream(self.stream):
                for bs in sets:
                    self.launch(pas, li, bs)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    for j in range(nl):
                        self.launch(pas, li, sets[j % nsets])
                g.replay()
                torch.cuda.synchronize()
                e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e_a.record(self.stream)
                for _ in range(reps):
                    g.replay()
                e_b.record(self.stream)
            torch.cuda.synchronize()
            mean_ms = e_a.elapsed_time(e_b) / (reps * nl)
            del g, sets
            nbytes = pass_bytes(L, pas, self.eb)
            info = self.plans[li][pas].describe()
            kt.append(dict(layer=L.name, pass_=pas, ms=mean_ms, bytes=nbytes, gbs=nbytes / (mean_ms * 1e-3) / 1e9,
                           li=li, variant=info["variant_name"], grid=info["grid"], block=info["block"],
                           shape=f"{L.c}x{L.h}x{L.w}/s{L.s}"))
        return kt

    def step_bytes(self):
        return step_bytes(self.layers, self.eb, self.fused)

    def plans_note(self):
        if not self.tuned:
            return "planner defaults"
        ch = sum(1 for t in self.tuned.values() for v in t.values() if v["index"] > 0)
        return (f"measured selection (tune.py, before the timed region): {ch} of "
                f"{sum(len(t) for t in self.tuned.values())} tuned passes changed")


def b128_workload(torch, dev, dtype, layout, steps, peak):
    """One entry of the >= 70 %-of-HBM target set (alpha 1.0 / 224, batch 128), same harness."""
    wl = Workload(torch, dev, 0, 1.0, 224, 128, dtype, layout)
    ms, per = wl.timed_steps(steps, 5)
    gbs = wl.step_bytes() / (ms / 1e3) / 1e9
    kt = wl.kernel_times(3)
    slow = min(kt, key=lambda k: k["gbs"] / 1.0)
    out = {"workload": workload_name(1.0, 224), "batch": 128, "dtype": dtype, "layout": layout, "steps": steps,
           "value": 128 / (ms / 1e3), "unit": "images/s", "ms_per_step": ms,
           "step_ms": {"p10": pct(per, 10), "p50": pct(per, 50), "p90": pct(per, 90)},
           "hbm_gbs": gbs, "frac_of_measured_peak": gbs / peak, "frac_of_8tbs": gbs / NOMINAL_HBM_GBS,
           "lowest_kernel": {"kernel": f"{slow['layer']}/{slow['pass_']}", "gbs": slow["gbs"],
                             "frac": slow["gbs"] / peak},
           "plans": wl.plans_note()}
    del wl
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_1803_09926_b200 import dp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.one_device:  # test mode: every rank on cuda:0 (NCCL refuses that; use --dist-backend gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    strong = args.global_batch > 0
    if strong:
        _, batch = dp.shard_batch(args.global_batch, world, rank)
        total_images = args.global_batch
    else:
        batch = args.batch
        total_images = args.batch * world
    peak, peak_src = hbm_peak()

    wl = Workload(torch, dev, rank, args.alpha, args.res, batch, args.dtype, args.layout, args.fused,
                  tune=not args.no_tune, plans_file=args.plans, serial=args.serial, graph=not args.no_graph)
    allreduce = (lambda: wl.bucket.allreduce()) if world > 1 else None
    barrier = (lambda: dist.barrier()) if world > 1 else None

    # ---- timed region: K steps, barrier + sync on both sides, CUDA events on the launching stream
    sampler = ClockSampler(local)
    sampler.start()
    ms_local, per = wl.timed_steps(args.steps, args.warmup, allreduce, barrier)
    sampler.stop()
    if world > 1:
        dist.barrier()
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_images / (ms / 1000.0)
    sbytes_local = wl.step_bytes()
    sb = torch.tensor([float(sbytes_local)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(sb)
    sbytes = int(sb.item())
    hbm_gbs = sbytes / (ms / 1000.0) / 1e9

    # ---- the all-reduce alone (N > 1): its time, bus bandwidth, NVLink-roofline fraction
    comm = None
    if world > 1:
        with torch.cuda.stream(wl.stream):
            for _ in range(5):
                wl.bucket.allreduce()
            torch.cuda.synchronize()
            dist.barrier()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(wl.stream)
            for _ in range(50):
                wl.bucket.allreduce()
            c1.record(wl.stream)
        torch.cuda.synchronize()
        ar_us = c0.elapsed_time(c1) * 1e3 / 50
        t = torch.tensor([ar_us], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ar_us = float(t.item())
        busbw = 2.0 * (world - 1) / world * wl.bucket.nbytes / (ar_us * 1e-6) / 1e9
        comm = {"allreduce_us": ar_us, "bytes": wl.bucket.nbytes, "bus_gbs": busbw,
                "nvlink_frac": busbw / NVLINK_GBS_PER_DIR, "share_of_step": ar_us * 1e-3 / ms,
                "backend": args.dist_backend + (" (test mode: every rank on cuda:0)" if args.one_device else ""),
                "nccl_algo": os.environ.get("NCCL_ALGO", "auto"), "nccl_proto": os.environ.get("NCCL_PROTO", "auto"),
                "note": "latency-bound: 178,560 B per step (SURVEY §8(e))"}

    kt = wl.kernel_times(args.kernel_reps) if args.kernel_reps > 0 else []
    kernel_sum_ms = sum(k["ms"] for k in kt)
    dom = max(kt, key=lambda k: k["ms"]) if kt else dict(layer="-", pass_="-", ms=float("nan"), bytes=0,
                                                         gbs=float("nan"))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tr = json.load(f)
            key = f"{args.alpha:g}/{args.res}/{batch}/{args.dtype}/{args.layout}/{dom['layer']}/{dom['pass_']}"
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
        s0 = wl.sets[0]
        host_in = [(b["x"].cpu().pin_memory(), b["dy"].cpu().pin_memory(), w.cpu().pin_memory())
                   for b, w in zip(s0, wl.w)]
        host_dw = torch.empty(wl.bucket.flat.shape, dtype=torch.float32).pin_memory()
        h2d = sum(t.numel() * t.element_size() for tup in host_in for t in tup)
        d2h = host_dw.numel() * 4

        def e2e_step():
            for b, w, (hx, hdy, hw) in zip(s0, wl.w, host_in):
                b["x"].copy_(hx, non_blocking=True)
                b["dy"].copy_(hdy, non_blocking=True)
                w.copy_(hw, non_blocking=True)
            wl.step_kernels(0)
            if world > 1:
                wl.bucket.allreduce()
            host_dw.copy_(wl.bucket.flat, non_blocking=True)

        with torch.cuda.stream(wl.stream):
            e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(wl.stream)
            for _ in range(args.e2e_steps):
                e2e_step()
            f1.record(wl.stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": total_images / (e2e_ms / 1000.0), "unit": "images/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": args.e2e_steps,
               "path": "python binding -> C ABI eager calls; pinned host->device copies of x, dy, w for all "
                       "13 layers and device->host copy of the dw bucket inside the timed region"}

    gpu_launches = len(wl.kernel_list()) * args.steps * world  # every rank launches the same step
    plans_note = wl.plans_note()
    footprint = wl.footprint
    nfused = sum(wl.fused)
    del wl
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---- the >= 70 % target set at batch 128 (N=1 only; each its own tuned, graph-replayed step)
    b128 = None
    if world == 1 and not args.no_b128 and not args.plans:
        b128 = [b128_workload(torch, dev, dt, lay, args.b128_steps, peak) for dt, lay in B128_SET]

    # ---- CPU baseline (oracle), rank 0 at N=1 only
    cpu = cpu_all = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu, cpu_all = cpu_baselines(layers_for(args.alpha, args.res, 1), args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded torch U[-1,1] on device; parity tests use the splitmix64 generator)",
            "config": {"workload": workload_name(args.alpha, args.res), "global_batch": total_images,
                       "batch_per_gpu": batch, "layers": 13, "layout": args.layout, "parallelism": f"dp{world}",
                       "l2": f"no flush: two input sets alternate between steps, each step's footprint "
                             f"{footprint / Workload.NSETS / 1e9:.2f} GB >> 126 MB L2",
                       "graph": not args.no_graph,
                       "schedule": ("serial" if args.serial else "bwd_filter on a side stream (overlaps bwd_data)") +
                                   f"; fused backward on {nfused}/13 layers",
                       "plans": plans_note, "dev_env": dev_env()},
            "step_ms": {"p10": pct(per, 10), "p50": pct(per, 50), "p90": pct(per, 90), "mean": ms_local},
            "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / world / peak, "hbm_frac_of_8tbs": hbm_gbs / world / NOMINAL_HBM_GBS,
            "algorithmic_bytes_per_step": sbytes,
            "roofline": ({"bound": "hbm", "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                          "frac": dom["gbs"] / peak, "traffic": traffic, "peak_source": peak_src,
                          "kernel": f"{dom['layer']}/{dom['pass_']}", "ms": dom["ms"], "bytes": dom["bytes"],
                          "timing": "back-to-back graph launches over rotating copies >= 2x L2"} if kt else None),
            "passes": passes,
            "kernel_sum_ms": kernel_sum_ms,
            "clocks": sampler.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "cpu_baseline_all_cores": cpu_all,
            "comm": comm,
            "workloads_b128": b128,
            "gpu_launches": gpu_launches,
            "paper_context": {"img_s": PAPER_CONTEXT_IMG_S, "hw": "GTX 1080 Ti, Caffe, Table III (context only)"},
        }
        if args.extra:
            line["kernels"] = [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in kk.items()} for kk in kt]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

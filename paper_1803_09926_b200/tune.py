"""Measurement-driven plan selection for the NCHW chunk kernels (a "find" step).

The planner in ``csrc/nchw_plan.cu`` scores chunk shapes with a cost model;
on B200 the best launch shape of a memory-bound stencil also depends on DRAM
page locality, L2 behaviour and ramp/tail effects the model does not see (a
sweep of dw2 bwd_filter spans 42-120 us over shapes the model ranks close).
``tune_layer`` times every candidate the library offers
(``dwconv_plan_candidates``) on the caller's tensors through immutable plan
handles (``dwconv_plan_create``) and returns the fastest as a plan per pass; it
changes no process-wide state (``install=True`` additionally installs the pick
with ``dwconv_plan_select`` for callers of the descriptor API).  Host-side
orchestration only: every launch it times is the library's own kernel; nothing
here computes a result.

Timing follows bench.py: back-to-back launches from a CUDA graph, cycling over
copies of the pass's tensors whose footprint is >= 2x L2, CUDA events on the
launching stream.  A candidate replaces the planner's default only if it is
faster by more than ``min_gain``.
"""
from __future__ import annotations

from typing import Dict, List, Optional

import torch

from . import ops
from ._lib import PASS_BWD, PASS_BWD_DATA, PASS_BWD_FILTER, PASS_FWD

PASSES = {"fwd": PASS_FWD, "bwd_data": PASS_BWD_DATA, "bwd_filter": PASS_BWD_FILTER, "bwd": PASS_BWD}


def _graph_us(calls, reps: int, stream: torch.cuda.Stream) -> float:
    # the tensor copies and the zero-filled workspace were made on the caller's
    # stream: order the timing stream after them (the bwd_filter tickets must
    # read as zero on the first launch)
    stream.wait_stream(torch.cuda.current_stream(stream.device))
    with torch.cuda.stream(stream):
        for c in calls:
            c()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for c in calls:
                c()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    del g
    return e0.elapsed_time(e1) * 1e3 / (reps * len(calls))


def tune_layer(d, x: torch.Tensor, dy: torch.Tensor, w: torch.Tensor, passes=("fwd", "bwd_data", "bwd_filter"),
               reps: int = 3, min_gain: float = 0.02, stream: Optional[torch.cuda.Stream] = None,
               install: bool = False) -> Dict[str, dict]:
    """Select the fastest candidate plan of each pass for descriptor ``d`` (NCHW or NHWC).

    x, dy, w: the layer's tensors (their values are not modified).  Returns, per pass, the chosen index,
    its time and the default's time (microseconds) and ``plan``: an ``ops.Plan`` of the pick (for passes
    with no candidate list: the planner's plan).
    """
    out: Dict[str, dict] = {}
    if d.n == 0:
        return out
    dev = x.device
    stream = stream or torch.cuda.Stream(device=dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    set_bytes = sum(t.numel() * t.element_size() for t in (x, dy)) * 2
    nsets = int(max(2, min(8, -(-2 * l2 // set_bytes))))
    sets = [dict(x=x, dy=dy)] + [dict(x=x.clone(memory_format=torch.preserve_format),
                                      dy=dy.clone(memory_format=torch.preserve_format)) for _ in range(nsets - 1)]
    for s in sets:
        s["y"] = torch.empty_like(dy)
        s["dx"] = torch.empty_like(x)
    dw = torch.empty(w.shape, dtype=torch.float32, device=dev)
    for name in passes:
        p = PASSES[name]
        cands: List[dict] = ops.dwconv_plan_candidates(d, p)
        if len(cands) <= 1:
            out[name] = {"index": 0 if cands else -1, "plan": ops.Plan(d, p, 0 if cands else -1),
                         "candidates": len(cands)}
            continue
        plans = [ops.Plan(d, p, i) for i in range(len(cands))]
        ws = None
        if p in (PASS_BWD_FILTER, PASS_BWD):
            ws = torch.zeros(max(16, max(pl.workspace_bytes for pl in plans)), dtype=torch.uint8, device=dev)

        def mk(pl, s):
            if p == PASS_FWD:
                return lambda: pl.fwd(s["x"], w, s["y"])
            if p == PASS_BWD_DATA:
                return lambda: pl.bwd_data(s["dy"], w, s["dx"])
            if p == PASS_BWD:
                return lambda: pl.bwd(s["x"], s["dy"], w, s["dx"], dw, ws)
            return lambda: pl.bwd_filter(s["x"], s["dy"], dw, ws)

        # two rounds: every candidate briefly, then the default and the 4 fastest
        # again with 4x the replays (the final pick is made on the second round)
        times = [_graph_us([mk(pl, s) for s in sets * 2], reps, stream) for pl in plans]
        finalists = sorted(set([0] + sorted(range(len(times)), key=lambda i: times[i])[:4]))
        for i in finalists:
            times[i] = _graph_us([mk(plans[i], s) for s in sets * 2], 4 * reps, stream)
        best = min(finalists, key=lambda i: times[i])
        if times[best] > times[0] * (1.0 - min_gain):
            best = 0
        if install:
            ops.dwconv_plan_select(d, p, best)
        out[name] = {"index": best, "us": times[best], "default_us": times[0], "candidates": len(cands),
                     "grid": cands[best]["grid"], "block": cands[best]["block"],
                     "planes_per_chunk": cands[best]["planes_per_chunk"],
                     "rows_per_band": cands[best]["rows_per_band"], "plan": plans[best]}
        del ws
    return out


def plans_from_selection(d, selection: Dict[str, dict]) -> Dict[str, "ops.Plan"]:
    """Plans for a selection returned by tune_layer (e.g. loaded from a file), without timing."""
    out = {}
    for name, r in selection.items():
        p = PASSES[name]
        idx = int(r["index"])
        if idx < 0:
            out[name] = ops.Plan(d, p, -1)
            continue
        cands = ops.dwconv_plan_candidates(d, p)
        if idx >= len(cands):
            raise RuntimeError(f"plan selection {name}:{idx} out of range ({len(cands)} candidates)")
        c = cands[idx]
        if "grid" in r and (c["grid"], c["block"]) != (r["grid"], r["block"]):
            raise RuntimeError(f"plan selection {name}:{idx} no longer matches the candidate list")
        out[name] = ops.Plan(d, p, idx)
    return out


def apply_selection(d, selection: Dict[str, dict]) -> None:
    """Install a selection process-wide (dwconv_plan_select) for callers of the descriptor API."""
    for name, pl in plans_from_selection(d, selection).items():
        if pl.candidate >= 0:
            ops.dwconv_plan_select(d, PASSES[name], pl.candidate)


def selection_json(tuned: Dict[str, dict]) -> Dict[str, dict]:
    """tune_layer's result without the plan objects (for --plans files)."""
    return {k: {kk: vv for kk, vv in v.items() if kk != "plan"} for k, v in tuned.items()}

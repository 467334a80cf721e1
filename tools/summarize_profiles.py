"""Summarise ncu captures (from tools/profile_round.sh) into profiles/<round>/.

* launch list: the last 39 dwconv launches of the bench run (``--kernel-reps 0``)
  are its last timed step, in step order (13 fwd, then bwd_data/bwd_filter per
  layer in reverse; the two backward kernels of a layer may appear in either
  order because bwd_filter runs on a side stream).  Writes a markdown table and profiles/ncu_traffic.json (DRAM bytes
  read+write per launch, keyed like bench.py's roofline lookup).
* full reports: key metrics of each ``full_<layer>_<pass>.ncu-rep``.

    python tools/summarize_profiles.py gpurun_out/prof r1 [--alpha 1 --res 224 --batch 64 --dtype f32 --layout nchw]
"""
import argparse
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem limit)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
]


def read_launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    iid, iname, imetric, ival = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = {}
    order = []
    for r in rows[1:]:
        k = int(r[iid])
        if k not in launches:
            launches[k] = {"name": r[iname]}
            order.append(k)
        launches[k][r[imetric]] = float(r[ival].replace(",", ""))
    return [launches[k] for k in order]


def to_bytes(v):
    return v  # launch list was captured with byte units (--csv keeps raw units)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("round")
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--layout", default="nchw")
    a = ap.parse_args()
    dst = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(dst, exist_ok=True)
    eb = 4 if a.dtype == "f32" else 2
    layers = synth.mobilenet_v1_dw(a.batch, a.alpha, a.res)
    step = [("fwd", L) for L in layers] + [(p, L) for L in reversed(layers) for p in ("bwd_data", "bwd_filter")]

    launches = [l for l in read_launches(os.path.join(a.src, "launches.csv"))
                if any(t in l["name"] for t in ("nchw_", "generic_", "dbf_kernel", "nhwc_", "small_", "band_", "lane_"))]

    def kind(name):
        import re as _re
        m = _re.search(r"(?:small_fd(?:_pair)?|lane_fd)_kernel<[^>]*,\s*(\d)>", name)
        if m:  # small-plane / lane-per-plane kernel: MODE 0 = fwd, 1 = bwd_data
            return "fwd" if m.group(1) == "0" else "bwd_data"
        if "small_fwd2_kernel" in name:
            return "fwd"
        if "small_bd2_kernel" in name:
            return "bwd_data"
        if "fwd_kernel" in name or "generic_fwd" in name:
            return "fwd"
        if "bwd_data" in name:
            return "bwd_data"
        return "bwd_filter"
    # the streams interleave under ncu's serialisation: take the last 13 launches of each
    # pass; within a pass the order is fixed (fwd: layer order, backward: reverse order)
    per = {k: [l for l in launches if kind(l["name"]) == k][-len(layers):] for k in ("fwd", "bwd_data", "bwd_filter")}
    last = []
    for (pas, L) in step:
        idx = [i for i, (p2, _) in enumerate(step) if p2 == pas].index(step.index((pas, L)))
        last.append(per[pas][idx])
    tot = sum(l["gpu__time_duration.sum"] for l in last)
    md = ["# ncu launch list — one bench step (per-kernel timing pass, serialised, cold-ish cache)", "",
          f"workload: MobileNet-v1 a{a.alpha:g} r{a.res} batch {a.batch} {a.dtype} {a.layout}; "
          f"`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`",
          "", "| # | layer | pass | kernel | ncu µs | share | DRAM MB (r+w) | algorithmic MB | GB/s (algorithmic/ncu time) |",
          "|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for i, ((pas, L), l) in enumerate(zip(step, last)):
        t_ns = l["gpu__time_duration.sum"]
        dram = l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
        alg = (L.x_elems() + L.y_elems()) * eb + (L.w_elems() * eb if pas != "bwd_filter" else L.w_elems() * 4)
        import re
        mm = re.search(r"(nchw_\w+_kernel|nhwc_\w+_kernel|small_\w+_kernel|band_\w+_kernel|lane_\w+_kernel|s?dbf_kernel|generic_\w+)<([^>]*)>",
                       l["name"])
        name = f"{mm.group(1)}<{mm.group(2)}>" if mm else l["name"][:40]
        md.append(f"| {i} | {L.name} | {pas} | {name} | {t_ns / 1e3:.2f} | {100 * t_ns / tot:.1f}% | {dram / 1e6:.1f} | "
                  f"{alg / 1e6:.1f} | {alg / t_ns:.0f} |")
        traffic[f"{a.alpha:g}/{a.res}/{a.batch}/{a.dtype}/{a.layout}/{L.name}/{pas}"] = dram
    md += ["", f"sum of launch times: {tot / 1e3:.1f} µs (serialised; the bench step overlaps launches)"]
    open(os.path.join(dst, "launch_list.md"), "w").write("\n".join(md) + "\n")
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1, sort_keys=True)

    reps = [(r, os.path.basename(r)[5:-8]) for r in sorted(glob.glob(os.path.join(a.src, "full_*.ncu-rep")))]
    reps += [(r, os.path.basename(r)[4:-4]) for r in sorted(glob.glob(os.path.join(a.src, "raw_*.csv")))]
    for rep, tag in reps:
        if rep.endswith(".csv"):  # raw page exported on the GPU box (ncu -i ... --page raw --csv)
            out = open(rep).read()
        else:
            out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if len(rows) < 3:
            continue  # capture failed (no matching launch)
        h, u, v = rows[0], rows[1], rows[2]
        d = {h[i]: (v[i], u[i]) for i in range(len(h))}
        md = [f"# ncu --set full: {tag} ({d.get('Kernel Name', ('?',))[0][:120]})", "",
              "| metric | value |", "|---|---|"]
        for k, label in KEYS:
            if k in d:
                md.append(f"| {label} (`{k}`) | {d[k][0]} {d[k][1]} |")
        stalls = sorted(((k, float(x[0].replace(",", ""))) for k, x in d.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled") and x[0] not in ("", "n/a")),
                        key=lambda t: -t[1])[:8]
        md += ["", "top stall samples:", ""] + [f"* `{k}`: {x:.0f}" for k, x in stalls]
        open(os.path.join(dst, f"ncu_{tag}.md"), "w").write("\n".join(md) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()

"""Print default-vs-best tables from tools/sweep_candidates.py JSON files (markdown).

The roofline column follows SURVEY §8(d) d.3: 7x7 (both dtypes) and bf16 5x5 are FP32-ALU bound and are
reported as useful FMA/s over the FP32 FMA peak (148 SMs x 128 FMA/clk x 1.965 GHz = 37.2 T FMA/s); every
other shape is HBM bound and reported against the measured copy peak."""
import json
import sys

for f in sys.argv[1:]:
    rows = json.load(open(f))
    best, dflt = {}, {}
    for r in rows:
        s = r["shape"]
        key = (f"m{s['m']} K{s['K']} s{s['s']} C{s['C']} {s['H']}x{s['W']} N{s['N']}", r["pass_"])
        if key not in best or r["us"] < best[key]["us"]:
            best[key] = r
        if r["candidate"] == 0:
            dflt[key] = r
    print(f"\n### {f} ({rows[0]['dtype']}, {rows[0]['layout']})\n")
    print("| shape | pass | default kernel | µs | bound | frac of roofline | useful TFMA/s | best candidate | µs |")
    print("|---|---|---|---|---|---|---|---|---|")
    for k in sorted(best):
        d, b = dflt[k], best[k]
        bn = b["variant"] + (f" S={b['S']} CB={b['CB']}" if b.get("S") else "")
        K = d["shape"]["K"]
        alu = K == 7 or (K == 5 and d["dtype"] == "bf16")
        frac = d["useful_tfma"] / 37.2 if alu else d["frac"]
        print(f"| {k[0]} | {k[1]} | {d['variant']} | {d['us']:.1f} | {'fp32 FMA' if alu else 'HBM'} | {frac:.2f} | "
              f"{d['useful_tfma']:.1f} | {bn} | {b['us']:.1f} |")

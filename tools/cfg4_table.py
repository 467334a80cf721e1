"""Print default-vs-best tables from tools/sweep_candidates.py JSON files (markdown)."""
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
    print("| shape | pass | default kernel | µs | frac of copy peak | useful TFMA/s | best candidate | µs |")
    print("|---|---|---|---|---|---|---|---|")
    for k in sorted(best):
        d, b = dflt[k], best[k]
        bn = b["variant"] + (f" S={b['S']} CB={b['CB']}" if b.get("S") else "")
        print(f"| {k[0]} | {k[1]} | {d['variant']} | {d['us']:.1f} | {d['frac']:.2f} | {d['useful_tfma']:.1f} | {bn} | {b['us']:.1f} |")

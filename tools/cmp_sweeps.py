"""Compare two sweep_candidates.py JSON files: default (candidate 0) and best candidate per shape/pass."""
import json
import sys


def load(p):
    out = {}
    for r in json.load(open(p)):
        s = r["shape"]
        key = (f"N{s['N']} C{s['C']} {s['H']}x{s['W']} K{s['K']} s{s['s']} m{s['m']}", r["pass_"])
        out.setdefault(key, []).append(r)
    return out


a, b = load(sys.argv[1]), load(sys.argv[2])
print(f"{'shape':32s} {'pass':10s} | {'A def':>7s} {'A best':>7s} | {'B def':>7s} {'B best':>7s} | best frac A -> B")
for k in a:
    if k not in b:
        continue
    ra, rb = a[k], b[k]
    ba, bb = min(ra, key=lambda r: r["us"]), min(rb, key=lambda r: r["us"])
    print(f"{k[0]:32s} {k[1]:10s} | {ra[0]['us']:7.1f} {ba['us']:7.1f} | {rb[0]['us']:7.1f} {bb['us']:7.1f} | "
          f"{ba['frac']:.2f} -> {bb['frac']:.2f}")

"""Split an ncu --page source --csv (SASS) dump into regions and sum the stall samples of each.

Regions: prologue (before the first FFMA/FFMA2), main loop (first..last FFMA), epilogue (after).
Also lists the top instructions by samples.
    python tools/src_regions.py gpurun_out/r3/src_bf_0.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
ins = [(r[isrc].strip(), int(r[isamp] or 0), int(r[iex] or 0)) for r in rows[2:] if len(r) > isamp]
fi = [i for i, (s, _, _) in enumerate(ins) if s.split()[0].startswith("FFMA") or (len(s.split()) > 1 and s.split()[1].startswith("FFMA"))]
tot = sum(x[1] for x in ins)
a, b = fi[0], fi[-1]
reg = {"prologue": ins[:a], "main": ins[a:b + 1], "epilogue": ins[b + 1:]}
for k, v in reg.items():
    print(f"{k:9s} samples {sum(x[1] for x in v):6d} ({100 * sum(x[1] for x in v) / tot:4.1f}%)  warp-instr {sum(x[2] for x in v)}")
print("top instructions:")
for s, n, e in sorted(ins, key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {n:5d} {e:9d}  {s[:90]}")

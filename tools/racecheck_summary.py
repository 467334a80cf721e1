"""Summarise a compute-sanitizer racecheck log: hazards grouped by (kind, kernel, source lines).

    compute-sanitizer --tool racecheck --print-limit 10000000 python tools/sanitize_cases.py 2>&1 | \
        python tools/racecheck_summary.py > summary.txt
"""
import collections
import re
import sys

txt = sys.stdin.read()
blocks = re.split(r"========= (?:Error|Warning): ", txt)[1:]
groups = collections.Counter()
for b in blocks:
    kind = b.split(" hazard")[0].strip()
    acc = re.findall(r"(Write|Read) Thread \S+ at (?:void )?(.+?)\+0x[0-9a-f]+ in (\S+)", b)
    kern = "?"
    if acc:
        m = re.search(r"(\w+)<", acc[0][1])
        kern = m.group(1) if m else acc[0][1][:60]
    groups[(kind, kern, tuple(f"{a}@{f}" for a, _, f in acc))] += 1
summ = re.findall(r"RACECHECK SUMMARY: .*", txt)
cases = re.findall(r"^(\w+): ok$", txt, re.M)
print(f"cases run: {', '.join(cases)}")
print(summ[-1] if summ else "no summary line")
print(f"distinct hazard sites: {len(groups)}")
for (kind, kern, acc), n in groups.most_common():
    print(f"{n:8d}  {kind:14s} {kern:28s} {'  '.join(acc)}")

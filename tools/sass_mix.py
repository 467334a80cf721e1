"""Opcode mix of one kernel's hot region (first to last FFMA2/FFMA) from an object file.

    python tools/sass_mix.py paper_1803_09926_b200/_build/nchw_fwd.cu.o 'nchw_fwd_kernelI13__nv_bfloat16Li3ELi1ELi7ELi8ELb1ELb0E'
"""
import re
import subprocess
import sys
from collections import Counter


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    names = re.findall(r"Function : (\S+)", subprocess.run(["cuobjdump", "-sass", obj], capture_output=True,
                                                            text=True).stdout)
    names = [n for n in names if re.search(pat, n)]
    for fn in names[:4]:
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
        ops = []
        for line in sass.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops.append(m.group(2))
        idx = [i for i, o in enumerate(ops) if o.startswith("FFMA")]
        if not idx:
            continue
        hot = ops[idx[0]:idx[-1] + 1]
        c = Counter(hot)
        print(f"== {fn[:140]}\n   hot region {len(hot)} instr of {len(ops)}; " +
              " ".join(f"{k}:{v}" for k, v in c.most_common(18)))


if __name__ == "__main__":
    main()

"""compute-sanitizer probe for one tcgen05 block-diagonal candidate (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1803_09926_b200 import ops
from paper_1803_09926_b200._lib import BF16, NHWC
shape = [int(v) for v in sys.argv[1].split(",")]
want = int(sys.argv[2])
N, C, H, W, K = shape
d = ops.make_desc(N, C, H, W, 1, K, 1, (K - 1) // 2, NHWC, BF16)
x = torch.randn(N, C, H, W, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
w = torch.randn(C, K, K, device="cuda").bfloat16()
y = torch.empty_like(x)
cands = ops.dwconv_plan_candidates(d, 0)
idx = [i for i, c in enumerate(cands) if c["variant_name"] == "nhwc_bdmma"]
i = idx[want]
c = cands[i]
print("cand", i, "S", c["planes_per_chunk"], "CB", c["rows_per_band"], "grid", c["grid"], flush=True)
ops.Plan(d, 0, i).fwd(x, w, y)
torch.cuda.synchronize()
print("done")

"""One rank of the gloo data-parallel tests (tests/test_dp.py): computes the filter
gradients of its batch shard, packs them in a DwBucket, all-reduces, and rank 0
saves the bucket.

    RANK=r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tests/dp_worker.py OUT.npy BATCH [MODE]

MODE ``oracle`` (default, CPU): each shard's dw from the oracle (test
infrastructure).  MODE ``cuda`` / ``cuda-int``: the product path on cuda:0 --
``dwconv_bwd_filter`` (C ABI) writes each layer's dw of the rank's shard
straight into the CUDA bucket views, then ``DwBucket.allreduce`` (gloo over CUDA
tensors; both ranks share the one GPU, which NCCL does not allow) -- on uniform
or small-integer inputs.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1803_09926_b200 import dp  # noqa: E402

LAYERS = [  # small layers with every shape feature the bucket must carry
    synth.Layer("a", 0, 4, 9, 9, k=3, s=1, p=1, m=1),
    synth.Layer("b", 0, 3, 10, 10, k=5, s=2, p=2, m=2),
    synth.Layer("c", 0, 5, 7, 7, k=3, s=2, p=1, m=3),
]


MOBILENET = [L for L in synth.mobilenet_v1_dw(0) if L.name in ("dw2", "dw4", "dw14", "dw24", "dw26")]


def global_inputs(L, i, batch, kind="unif"):
    if kind == "int":
        x = synth.integers(synth.layer_seed(i, "x"), (batch, L.c, L.h, L.w), 2)
        dy = synth.integers(synth.layer_seed(i, "dy"), (batch, L.c * L.m, L.ho, L.wo), 2)
    else:
        x = synth.uniform(synth.layer_seed(i, "x"), (batch, L.c, L.h, L.w))
        dy = synth.uniform(synth.layer_seed(i, "dy"), (batch, L.c * L.m, L.ho, L.wo))
    return x, dy


def cuda_shard_dw(layers, bucket, start, count, batch, kind):
    from paper_1803_09926_b200 import ops
    from paper_1803_09926_b200._lib import F32, NCHW
    for i, L in enumerate(layers):
        x, dy = global_inputs(L, i, batch, kind)
        xs = torch.from_numpy(np.ascontiguousarray(x[start:start + count], dtype=np.float32)).cuda()
        dys = torch.from_numpy(np.ascontiguousarray(dy[start:start + count], dtype=np.float32)).cuda()
        d = ops.make_desc(count, L.c, L.h, L.w, L.m, L.k, L.s, L.p, NCHW, F32)
        ws = torch.zeros(max(16, ops.dwconv_bwd_filter_workspace_bytes(d)), dtype=torch.uint8, device="cuda")
        ops.dwconv_bwd_filter(d, xs, dys, bucket.views[i], ws)
    torch.cuda.synchronize()


def main():
    out, batch = sys.argv[1], int(sys.argv[2])
    mode = sys.argv[3] if len(sys.argv) > 3 else "oracle"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    start, count = dp.shard_batch(batch, world, rank)
    if mode == "oracle":
        bucket = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in LAYERS], device="cpu")
        for i, L in enumerate(LAYERS):
            x, dy = global_inputs(L, i, batch)
            dwv, _ = oracle.bwd_filter(x[start:start + count], dy[start:start + count], (L.c * L.m, L.k, L.k),
                                       L.s, L.p)
            bucket.views[i].copy_(torch.from_numpy(dwv.astype(np.float32)))
    else:
        torch.cuda.set_device(0)
        layers = LAYERS + MOBILENET
        bucket = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in layers], device="cuda")
        bucket.flat.fill_(float("nan"))  # every view must be overwritten (padding re-zeroed below)
        for i, L in enumerate(layers):
            o, n = bucket.offsets[i], L.c * L.m * L.k * L.k
            nxt = bucket.offsets[i + 1] if i + 1 < len(layers) else bucket.numel
            bucket.flat[o + n:nxt].zero_()
        cuda_shard_dw(layers, bucket, start, count, batch, "int" if mode == "cuda-int" else "unif")
    bucket.allreduce()
    if rank == 0:
        np.save(out, bucket.flat.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""One rank of the gloo data-parallel test (tests/test_dp.py): computes the filter
gradients of its batch shard with the oracle (test infrastructure), packs them in
a DwBucket, all-reduces, and rank 0 saves the bucket.

    RANK=r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tests/dp_worker.py OUT.npy BATCH
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


def global_inputs(L, i, batch):
    x = synth.uniform(synth.layer_seed(i, "x"), (batch, L.c, L.h, L.w))
    dy = synth.uniform(synth.layer_seed(i, "dy"), (batch, L.c * L.m, L.ho, L.wo))
    return x, dy


def main():
    out, batch = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    start, count = dp.shard_batch(batch, world, rank)
    bucket = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in LAYERS], device="cpu")
    for i, L in enumerate(LAYERS):
        x, dy = global_inputs(L, i, batch)
        dwv, _ = oracle.bwd_filter(x[start:start + count], dy[start:start + count], (L.c * L.m, L.k, L.k), L.s, L.p)
        bucket.views[i].copy_(torch.from_numpy(dwv.astype(np.float32)))
    bucket.allreduce()
    if rank == 0:
        np.save(out, bucket.flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Data-parallel dw all-reduce, CPU/gloo world_size 2.

The global dw is the batch sum of Eq. 4, so
sharding the batch over ranks and SUM-all-reducing the per-rank dw must give the
full-batch dw.  The per-rank dw come from the oracle here (no GPU); the GPU test
checks the same identity through the CUDA path on one device.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from dp_worker import LAYERS, MOBILENET, global_inputs  # noqa: E402

from paper_1803_09926_b200 import dp  # noqa: E402


def test_shard_batch_tiles_the_batch():
    for batch in (0, 1, 2, 5, 64, 129):
        for world in (1, 2, 3, 8):
            got = [dp.shard_batch(batch, world, r) for r in range(world)]
            assert sum(c for _, c in got) == batch
            pos = 0
            for s, c in got:
                assert s == pos and c >= 0
                pos += c
            assert max(c for _, c in got) - min(c for _, c in got) <= 1
    with pytest.raises(ValueError):
        dp.shard_batch(4, 2, 2)


def test_bucket_layout():
    L = synth.mobilenet_v1_dw(1)
    b = dp.DwBucket([(l.c * l.m, l.k, l.k) for l in L], device="cpu")
    assert b.numel == 44640 and b.nbytes == 178560  # SURVEY §8(a) a6 for alpha 1.0
    for v, o in zip(b.views, b.offsets):
        assert o % dp.ALIGN_ELEMS == 0
        assert v.data_ptr() == b.flat.data_ptr() + 4 * o
    b.views[3].fill_(2.0)
    assert float(b.flat.sum()) == 2.0 * b.views[3].numel()
    b.zero_()
    assert float(b.flat.abs().sum()) == 0.0
    assert b.allreduce() is None  # no process group: no-op


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_world2(out, batch, mode="oracle"):
    env = dict(os.environ, WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dp_worker.py"), out, str(batch), mode],
                              env=dict(env, RANK=str(r)), stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=180)[0].decode())
        except subprocess.TimeoutExpired:
            p.kill()
            raise
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    return np.load(out)


@pytest.mark.parametrize("batch", [6, 5, 1])  # even, ragged, one rank empty
def test_gloo_world2_allreduce_equals_full_batch(tmp_path, batch):
    flat = _run_world2(str(tmp_path / "bucket.npy"), batch)
    ref = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in LAYERS], device="cpu")
    for i, L in enumerate(LAYERS):
        x, dy = global_inputs(L, i, batch)
        dwv, absum = oracle.bwd_filter(x, dy, (L.c * L.m, L.k, L.k), L.s, L.p)
        got = flat[ref.offsets[i]:ref.offsets[i] + dwv.size].reshape(dwv.shape)
        # fp32 parity bound plus one fp32 rounding per rank's partial
        tol = 1e-5 * absum + 1e-7
        assert np.all(np.abs(got - dwv) <= tol), (L, np.max(np.abs(got - dwv) - tol))
    # padding between layers stays zero
    mask = np.ones(flat.size, bool)
    for i, L in enumerate(LAYERS):
        mask[ref.offsets[i]:ref.offsets[i] + L.c * L.m * L.k * L.k] = False
    assert np.all(flat[mask] == 0)


@pytest.mark.gpu
def test_gpu_batch_shards_sum_to_full_batch():
    """One device, two 'ranks': dw(shard 0) + dw(shard 1) == dw(full batch) (integer inputs: exact)."""
    import torch
    import paper_1803_09926_b200 as dwl
    for L in synth.mobilenet_v1_dw(5)[:4]:
        x = torch.from_numpy(synth.integers(11, (L.n, L.c, L.h, L.w), 3).astype(np.float32)).cuda()
        dy = torch.from_numpy(synth.integers(12, (L.n, L.c, L.ho, L.wo), 3).astype(np.float32)).cuda()
        wshape = (L.c, L.k, L.k)
        full = dwl.bwd_filter(x, dy, wshape, L.s, L.p)
        bucket = dp.DwBucket([wshape], device="cuda")
        for r in range(2):
            s, c = dp.shard_batch(L.n, 2, r)
            bucket.views[0].add_(dwl.bwd_filter(x[s:s + c].contiguous(), dy[s:s + c].contiguous(), wshape, L.s, L.p))
        torch.cuda.synchronize()
        assert torch.equal(bucket.views[0], full), L


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["int", "unif"])
@pytest.mark.parametrize("batch", [6, 5])  # even, ragged
def test_gpu_world2_cuda_dw_allreduce_equals_oracle_global_batch(tmp_path, batch, kind):
    """Row a6 end to end through the product path (R6): two processes on one GPU, each runs
    dwconv_bwd_filter on its batch shard into the CUDA DwBucket, DwBucket.allreduce over gloo; the reduced
    bucket must equal the oracle's dw of the GLOBAL batch -- bitwise on small integers (P6/P8), within the
    fp32 bound plus one rounding per rank partial on uniform data (R6)."""
    flat = _run_world2(str(tmp_path / "bucket.npy"), batch, "cuda-int" if kind == "int" else "cuda")
    layers = LAYERS + MOBILENET
    ref = dp.DwBucket([(L.c * L.m, L.k, L.k) for L in layers], device="cpu")
    for i, L in enumerate(layers):
        x, dy = global_inputs(L, i, batch, kind)
        dwv, absum = oracle.bwd_filter(x, dy, (L.c * L.m, L.k, L.k), L.s, L.p)
        got = flat[ref.offsets[i]:ref.offsets[i] + dwv.size].reshape(dwv.shape)
        if kind == "int":
            assert np.array_equal(got, dwv.astype(np.float32)), L
        else:
            tol = 1e-5 * absum + 2 * 2.0 ** -24 * np.abs(dwv)
            assert np.all(np.abs(got - dwv) <= tol), (L, np.max(np.abs(got - dwv) - tol))
    mask = np.ones(flat.size, bool)
    for i, L in enumerate(layers):
        mask[ref.offsets[i]:ref.offsets[i] + L.c * L.m * L.k * L.k] = False
    assert np.all(flat[mask] == 0)

"""The seeded input generator and the layer catalog (CPU only)."""
import json
import os

import numpy as np

import synth


def test_generator_deterministic_and_in_range():
    a = synth.uniform(7, (3, 5, 4, 4))
    b = synth.uniform(7, (3, 5, 4, 4))
    assert np.array_equal(a, b) and a.dtype == np.float32
    assert a.min() >= -1.0 and a.max() <= 1.0
    assert not np.array_equal(a, synth.uniform(8, (3, 5, 4, 4)))
    assert synth.uniform(1, (0, 3, 2, 2)).size == 0


def test_splitmix64_reference_values():
    # splitmix64 with state 0: first outputs of the published generator (Vigna, 2015)
    z = synth.splitmix64(0, 0, 3)
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_batch_shard_equals_slice():
    shape = (8, 3, 5, 5)
    full = synth.uniform(3, shape)
    per = int(np.prod(shape[1:]))
    for r in range(4):
        part = synth.uniform(3, (2,) + shape[1:], start=2 * r * per)
        assert np.array_equal(part, full[2 * r:2 * r + 2])


def test_bf16_values_and_bits_roundtrip():
    a = synth.uniform(4, (1000,), "bf16")
    bits = synth.to_bf16_bits(a)
    assert np.array_equal(synth.from_bf16_bits(bits), a)
    # RNE ties-to-even at the bf16 boundary
    v = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8], dtype=np.float32)
    assert np.array_equal(synth._bf16_round_f32(v), np.array([1.0, 1.0 + 2.0 ** -6], dtype=np.float32))


def test_integer_sets():
    k = synth.integers(5, (10000,), 4)
    assert set(np.unique(k).tolist()) == set(range(-4, 5))


def test_catalog_matches_table3(golden_dir):
    with open(os.path.join(golden_dir, "table3_layers.json")) as f:
        g = json.load(f)
    layers = synth.mobilenet_v1_dw(g["batch"])
    assert len(layers) == len(g["layers"]) == 13
    for L, row in zip(layers, g["layers"]):
        assert L.name == f"dw{row['layer']}"
        assert (L.k, L.s, L.h, L.w, L.c, L.n) == (g["kernel"], row["stride"], row["hw"], row["hw"], row["c"], 64)
    # output sizes chain to the next layer's input at 224 px
    assert [L.ho for L in layers] == [112, 56, 56, 28, 28, 14, 14, 14, 14, 14, 14, 7, 7]


def test_catalog_reproduces_table1(golden_dir):
    """Table I: mult-add and parameter shares of MobileNet-v1 by layer type.

    The dw layers come from the catalog; the rest of the network (stem 3x3/2,
    pointwise 1x1 layers, FC 1024->1000) is rebuilt here from the same table.
    """
    with open(os.path.join(golden_dir, "table1_ratios.json")) as f:
        g = json.load(f)
    dw = synth.mobilenet_v1_dw(1)
    pw_out = [64, 128, 128, 256, 256, 512, 512, 512, 512, 512, 512, 1024, 1024]
    ma = {"dw3x3": sum(L.fma() for L in dw),
          "conv1x1": sum(L.c * co * L.ho * L.wo for L, co in zip(dw, pw_out)),
          "conv3x3": 112 * 112 * 32 * 3 * 9,
          "fc": 1024 * 1000}
    pa = {"dw3x3": sum(L.w_elems() for L in dw),
          "conv1x1": sum(L.c * co for L, co in zip(dw, pw_out)),
          "conv3x3": 32 * 3 * 9,
          "fc": 1024 * 1000}
    tma, tpa = sum(ma.values()), sum(pa.values())
    for k, v in g["params_pct"].items():
        assert abs(100.0 * pa[k] / tpa - v) < 0.01, k
    for k, v in g["mult_adds_pct"].items():
        got = 100.0 * ma[k] / tma
        if k == "conv3x3":  # printed 1.19, recomputed 1.91 (digit transposition)
            assert abs(got - 1.91) < 0.01 and abs(v - 1.19) < 1e-9
        else:
            assert abs(got - v) < 0.01, k
    assert pa["dw3x3"] == 44640  # the flat dw bucket


def test_width_resolution_variants():
    L = synth.mobilenet_v1_dw(128, alpha=0.25, resolution=128)
    assert [l.c for l in L][:3] == [8, 16, 32] and L[0].h == 64 and L[-1].h == 4
    L = synth.mobilenet_v1_dw(128, alpha=0.75, resolution=160)
    assert L[0].c == 24 and L[0].h == 80 and L[-1].c == 768 and L[-1].h == 5

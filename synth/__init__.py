"""Seeded synthetic inputs and the MobileNet-v1 depthwise layer catalog.

This module is shared by the oracle side (tests, ``bench.py --impl reference``)
and the CUDA side (tests, ``bench.py``).  It holds NONE of the method's
arithmetic: it only produces input values and workload shapes.  Both sides
receive the same arrays from here and nothing else is shared between them.

Generator (SPEC.md S:53-61 / S:70 "splitmix-style"):
counter-based splitmix64, ``value_i = mix(seed + (i + 1) * GOLDEN)`` where ``i``
is the element's LOGICAL NCHW flat index.  Because it is counter-based:

* the same logical tensor has the same values in NCHW and NHWC storage;
* a batch shard ``[n0, n1)`` equals the slice of the global tensor, for any
  number of data-parallel ranks.

Float draws are U[-1, 1] rounded once (RNE) to the storage dtype; integer draws
are uniform on ``{-a, ..., a}`` (the exact-parity value sets of SURVEY.md §8(c)
c.6).  The MobileNet-v1 catalog follows PAPER.md Table III for the
13 depthwise layers and the width/resolution multipliers of Table V.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """uint64 stream values for counters ``start .. start+count-1``."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _bf16_round_f32(a: np.ndarray) -> np.ndarray:
    """fp32 array -> fp32 array holding the RNE-to-bf16 value (finite inputs)."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def uniform(seed: int, shape: Sequence[int], dtype: str = "f32", start: int = 0) -> np.ndarray:
    """U[-1,1] values (logical C-order flat index), rounded to ``dtype`` storage.

    Returns float32 values (for ``bf16`` the float32 array holds exact bf16
    values).  ``start`` offsets the counter, which is how a batch shard is drawn.
    """
    n = int(np.prod(shape)) if len(shape) else 1
    z = splitmix64(seed, start, n)
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    v = (2.0 * u - 1.0).astype(np.float32)  # one RNE rounding double -> fp32
    if dtype == "bf16":
        v = _bf16_round_f32(v)
    elif dtype != "f32":
        raise ValueError(dtype)
    return v.reshape(shape)


def integers(seed: int, shape: Sequence[int], amax: int, start: int = 0) -> np.ndarray:
    """Uniform integers in ``{-amax..amax}`` as float32 (exact in fp32 and bf16 for amax<=256)."""
    n = int(np.prod(shape)) if len(shape) else 1
    z = splitmix64(seed, start, n)
    k = (z % np.uint64(2 * amax + 1)).astype(np.int64) - amax
    return k.astype(np.float32).reshape(shape)


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 array holding bf16-representable values -> uint16 bit patterns."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if np.any(b & np.uint32(0xFFFF)):
        raise ValueError("values are not bf16-representable")
    return (b >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(h: np.ndarray) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def nchw_to_nhwc(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a.transpose(0, 2, 3, 1))


def nhwc_to_nchw(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a.transpose(0, 3, 1, 2))


# --------------------------------------------------------------------------
# Workload catalog
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Layer:
    """One depthwise layer: input x is [n, c, h, w]; weights [c*m, k, k]."""
    name: str
    n: int
    c: int
    h: int
    w: int
    k: int = 3
    s: int = 1
    p: int = 1
    m: int = 1

    @property
    def ho(self) -> int:
        return (self.h + 2 * self.p - self.k) // self.s + 1

    @property
    def wo(self) -> int:
        return (self.w + 2 * self.p - self.k) // self.s + 1

    def x_elems(self) -> int:
        return self.n * self.c * self.h * self.w

    def y_elems(self) -> int:
        return self.n * self.c * self.m * self.ho * self.wo

    def w_elems(self) -> int:
        return self.c * self.m * self.k * self.k

    def fma(self) -> int:
        """Multiply-adds of one pass (the same for fwd, bwd_data, bwd_filter)."""
        return self.y_elems() * self.k * self.k

    def with_batch(self, n: int) -> "Layer":
        return dataclasses.replace(self, n=n)


# PAPER.md Table III: layer number, stride, input H=W, channels C.
MOBILENET_V1_DW: Tuple[Tuple[int, int, int, int], ...] = (
    (2, 1, 112, 32),
    (4, 2, 112, 64),
    (6, 1, 56, 128),
    (8, 2, 56, 128),
    (10, 1, 28, 256),
    (12, 2, 28, 256),
    (14, 1, 14, 512),
    (16, 1, 14, 512),
    (18, 1, 14, 512),
    (20, 1, 14, 512),
    (22, 1, 14, 512),
    (24, 2, 14, 512),
    (26, 1, 7, 1024),
)


def mobilenet_v1_dw(batch: int, alpha: float = 1.0, resolution: int = 224) -> List[Layer]:
    """The 13 depthwise 3x3 layers of MobileNet-v1 at width ``alpha`` and input ``resolution``.

    Spatial size scales as H * resolution / 224 (the stem halves 224 -> 112);
    channels as C * alpha (exact integers for alpha in {0.25, 0.5, 0.75, 1}).
    Padding is symmetric p=1 (reading R2).
    """
    out = []
    for num, s, h224, c in MOBILENET_V1_DW:
        h = (h224 * resolution) // 224
        cc = int(round(c * alpha))
        out.append(Layer(name=f"dw{num}", n=batch, c=cc, h=h, w=h, k=3, s=s, p=1, m=1))
    return out


def layer_seed(layer_index: int, tensor: str) -> int:
    """seed(layer L, tensor t) = 1000*L + {x:1, w:2, dy:3}."""
    return 1000 * layer_index + {"x": 1, "w": 2, "dy": 3}[tensor]

"""Data-parallel plumbing for the filter gradients.

Under data parallelism every rank runs the three depthwise passes on its own
slice of the global batch.  The filter gradient is a sum over the batch
(``dw[o,i,jj] = sum_n sum_{oh,ow} x * dy``; Eq. 4, and the
batch sum of SPEC S:342), so the global dw is the SUM over ranks of the per-rank
dw -- one all-reduce of every layer's dw.  ``DwBucket`` keeps all layers' dw
back to back in one flat fp32 buffer (44,640 floats = 178,560 B for MobileNet-v1
alpha 1.0), so a step issues exactly one collective (NCCL on B200, gloo in the
CPU tests).  fwd and bwd_data need no exchange at all.

Nothing here computes: the per-rank dw comes from ``dwconv_bwd_filter`` (C ABI),
the reduction from ``torch.distributed``.
"""
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

ALIGN_ELEMS = 32  # every layer's dw view starts on a 128-B boundary


def shard_batch(global_batch: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous batch slice ``[start, start + count)`` of ``rank``.

    The first ``global_batch % world`` ranks take one extra image, so the slices
    tile ``[0, global_batch)`` exactly (empty slices are allowed: a rank with no
    images contributes dw = 0, which ``dwconv_bwd_filter`` writes for N = 0).
    """
    if world < 1 or not 0 <= rank < world or global_batch < 0:
        raise ValueError(f"bad shard request: batch={global_batch} world={world} rank={rank}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


class DwBucket:
    """One flat fp32 buffer holding the dw of every layer.

    ``views[i]`` is layer i's ``[C*m, kh, kw]`` gradient (what ``dwconv_bwd_filter``
    overwrites); ``flat`` is what the all-reduce moves.
    """

    def __init__(self, wshapes: Sequence[Sequence[int]], device="cuda"):
        self.shapes = [tuple(int(v) for v in s) for s in wshapes]
        self.offsets: List[int] = []
        off = 0
        for s in self.shapes:
            self.offsets.append(off)
            n = 1
            for v in s:
                n *= v
            off += (n + ALIGN_ELEMS - 1) // ALIGN_ELEMS * ALIGN_ELEMS
        self.numel = off
        self.flat = torch.zeros(off, dtype=torch.float32, device=device)
        self.views = []
        for s, o in zip(self.shapes, self.offsets):
            n = 1
            for v in s:
                n *= v
            self.views.append(self.flat[o:o + n].view(*s))

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4

    def zero_(self) -> None:
        self.flat.zero_()

    def allreduce(self, group: Optional[dist.ProcessGroup] = None, average: bool = False, async_op: bool = False):
        """SUM the bucket over the ranks of ``group`` (in place); ``average`` divides by the group size.

        With ``async_op`` the work handle is returned (``average`` is then left
        to the caller).  A no-op when torch.distributed is not initialised or the
        group has one rank.
        """
        if not dist.is_available() or not dist.is_initialized():
            return None
        world = dist.get_world_size(group)
        if world == 1:
            return None
        work = dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
        if async_op:
            return work
        if average:
            self.flat.div_(world)
        return None

"""Data-parallel sharding of the sentence batch (north star (4)).

Sentences are independent (the training loop just sums
per-sentence GrammarGrads, train.py:206-218), so the batch is split across
ranks, every rank holds a full replica of the read-only L, R, root, and the
only exchange is ONE all-reduce (sum) of the grammar gradients
[dL | dR | droot] in a single flat fp32 buffer.  dunary and log_z stay
sharded.  One process per GPU; NCCL over NVLink in production, gloo in the
CPU tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) slice of n_items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_by_length(lengths, world: int, rank: int) -> list[int]:
    """Length-balanced sharding: sentences sorted by length, dealt round-robin
    so every rank gets a similar total chart size; returns sentence indices."""
    order = sorted(range(len(lengths)), key=lambda k: (-int(lengths[k]), k))
    return [k for pos, k in enumerate(order) if pos % world == rank]


class GradBucket:
    """A persistent flat buffer holding [dL | dR | droot] for one all-reduce."""

    def __init__(self, shapes, device, dtype=torch.float32):
        self.shapes = [torch.Size(s) for s in shapes]
        self.sizes = [s.numel() for s in self.shapes]
        self.flat = torch.empty(sum(self.sizes), dtype=dtype, device=device)

    def views(self):
        out, off = [], 0
        for shp, n in zip(self.shapes, self.sizes):
            out.append(self.flat[off:off + n].view(shp))
            off += n
        return out

    def pack(self, tensors):
        for dst, src in zip(self.views(), tensors):
            dst.copy_(src)

    def allreduce(self, group=None, async_op: bool = False):
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return None
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def allreduce_grads(tensors, group=None):
    """Sum `tensors` over ranks with a single collective; returns new tensors."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(tensors)
    bucket = GradBucket([t.shape for t in tensors], tensors[0].device, tensors[0].dtype)
    bucket.pack(tensors)
    bucket.allreduce(group)
    return bucket.views()

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


_BUCKETS: dict = {}


def allreduce_grads(tensors, group=None):
    """Sum `tensors` over ranks with a single collective on one flat buffer.

    The bucket is allocated once per (shapes, device, dtype) and reused, so
    the returned views are overwritten by the next call with the same
    shapes (the training step consumes them within the step)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(tensors)
    key = (tuple(tuple(t.shape) for t in tensors), str(tensors[0].device), tensors[0].dtype)
    bucket = _BUCKETS.get(key)
    if bucket is None:
        bucket = _BUCKETS[key] = GradBucket([t.shape for t in tensors], tensors[0].device,
                                            tensors[0].dtype)
    bucket.pack(tensors)
    bucket.allreduce(group)
    return bucket.views()


class DataParallelInside:
    """The data-parallel fwd + bwd step of the inside op.

    Each rank runs its shard of the sentence batch through the engine
    (fi_inside_forward + fi_inside_backward_ex) and the grammar gradients
    land directly in the views of ONE persistent flat bucket
    [dL | dR | droot] -- no packing copy.  The bucket is all-reduced in two
    chunks on a communication stream: dL as soon as the backward's dL-ready
    event fires (its all-reduce overlaps dR's weight-gradient GEMM), then
    [dR | droot] when the backward ends.  The same calls are captured into
    a CUDA graph by the caller (bench.py), NCCL included.  dunary and log_z
    stay sharded (per sentence).  This replaces the reference's
    sentence-sequential gradient sum (train.py:206-218)."""

    def __init__(self, n_nt: int, n_pt: int, batch: int, max_len: int, gemm_dtype: str = "bf16",
                 chart_dtype: str = "auto", device=None, group=None, slots: int = 1):
        from . import _lib
        self._lib = _lib
        self.lib = _lib.load()
        self.device = torch.device(device or "cuda")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.shape = _lib.shape(n_nt, n_pt, batch, max_len, gemm_dtype, False, chart_dtype)
        nbytes = _lib.workspace_bytes(self.shape)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        # output slots: a caller streaming results to the host alternates two
        # so step k's device->host copy overlaps step k+1 (bench.py e2e)
        self.slots = []
        for _ in range(max(1, slots)):
            bucket = GradBucket([(n_nt, n_nt + n_pt), (n_nt, n_nt + n_pt), (n_nt,)], self.device)
            dL, dR, droot = bucket.views()
            self.slots.append(dict(
                bucket=bucket, dL=dL, dR=dR, droot=droot,
                tail=bucket.flat[n_nt * (n_nt + n_pt):],                  # [dR | droot]
                log_z=torch.empty(batch, dtype=torch.float32, device=self.device),
                dunary=torch.empty(batch, max_len, n_pt, dtype=torch.float32,
                                   device=self.device)))
        self.bucket, self.dL, self.dR, self.droot, self.log_z, self.dunary = (
            self.slots[0][k] for k in ("bucket", "dL", "dR", "droot", "log_z", "dunary"))
        self.comm = torch.cuda.Stream(self.device) if self.world > 1 else None
        self.dl_ready = torch.cuda.Event()
        self.dl_ready.record(torch.cuda.current_stream(self.device))  # materialise the handle

    def step(self, L, R, root, unary, lengths, grad_log_z, slot: int = 0):
        """log_z (B,), dL, dR (N, N+P) and droot (N,) summed over ranks, dunary
        (B, l, P) of this rank's sentences, in output slot ``slot``.  Inputs as
        the op's (contiguous fp32 CUDA tensors, lengths int32);
        stream-ordered, no host sync."""
        import ctypes
        lib, _lib = self.lib, self._lib
        o = self.slots[slot]
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        cur = torch.cuda.current_stream(self.device)
        st = ctypes.c_void_p(cur.cuda_stream)
        sh = ctypes.byref(self.shape)
        _lib.check(lib.fi_inside_forward(sh, p(L), p(R), p(root), p(unary), p(lengths),
                                         p(o["log_z"]), p(self.ws), st))
        ev = ctypes.c_void_p(self.dl_ready.cuda_event) if self.world > 1 else ctypes.c_void_p(0)
        _lib.check(lib.fi_inside_backward_ex(
            sh, p(L), p(R), p(root), p(unary), p(lengths), p(o["log_z"]), p(grad_log_z),
            p(o["dL"]), p(o["dR"]), p(o["droot"]), p(o["dunary"]), p(self.ws), st, ev))
        if self.world > 1:
            with torch.cuda.stream(self.comm):
                self.comm.wait_event(self.dl_ready)
                dist.all_reduce(o["dL"], group=self.group)      # overlaps dR's wgrad GEMM
                self.comm.wait_stream(cur)
                dist.all_reduce(o["tail"], group=self.group)    # [dR | droot]
            cur.wait_stream(self.comm)
        return o["log_z"], o["dL"], o["dR"], o["droot"], o["dunary"]

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


class HostStreamedStep:
    """The op's step fed from host memory, the way a training loop calls it:
    every step brings new grammar tables and tokens from pinned host buffers
    and takes log Z and the GrammarGrad tables (dL, dR, droot, d_emit) back.

    The device part -- unary gather, ``DataParallelInside.step`` (engine
    fwd + bwd, all-reduce at N > 1) and the d_emit scatter
    (inside.py:420-423) -- is captured once per buffer slot as a CUDA graph
    over static device inputs; a step is then H2D (side stream) -> one
    graph replay -> D2H (side stream).  Two slots alternate, so step k+1's
    copies in and step k's copies out overlap the compute.  ``step`` only
    enqueues; ``synchronize`` waits for every copy."""

    def __init__(self, dpi: DataParallelInside, vocab: int, lengths, grad_log_z):
        self.dpi = dpi
        dev = dpi.device
        s = dpi.shape
        n, p, b, l = s.n_nt, s.n_pt, s.batch, s.max_len
        self.n_pt = p
        self.lengths, self.gvec = lengths, grad_log_z
        self.comp = torch.cuda.current_stream(dev)
        self.s_in = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        nslot = len(dpi.slots)
        self.inputs = [dict(L=torch.empty(n, n + p, device=dev), R=torch.empty(n, n + p, device=dev),
                            root=torch.empty(n, device=dev), emit=torch.empty(p, vocab, device=dev),
                            tok=torch.zeros(b, l, dtype=torch.int64, device=dev))
                       for _ in range(nslot)]
        self.in_ready = [torch.cuda.Event() for _ in range(nslot)]
        self.in_free = [None] * nslot
        self.out_ready = [torch.cuda.Event() for _ in range(nslot)]
        self.out_free = [None] * nslot
        self.outputs = [None] * nslot
        self.capture_error = False
        self.graphs = [self._capture(k) for k in range(nslot)]

    def _device_step(self, k):
        d = self.inputs[k]
        # inside.py:296-298; the (V, P) transpose first, so the row gather is
        # coalesced (53 -> 33 us at config 3)
        un = d["emit"].t().contiguous()[d["tok"]]
        log_z, dL, dR, droot, dun = self.dpi.step(d["L"], d["R"], d["root"], un, self.lengths,
                                                  self.gvec, slot=k)
        d_emit = torch.zeros(d["emit"].shape[1], self.n_pt, device=un.device).index_add_(
            0, d["tok"].view(-1), dun.reshape(-1, self.n_pt))        # inside.py:420-423
        return dL, dR, droot, d_emit.t(), log_z

    def _capture(self, k):
        side = torch.cuda.Stream(self.dpi.device)
        side.wait_stream(self.comp)
        with torch.cuda.stream(side):
            for _ in range(2):
                self._device_step(k)
        self.comp.wait_stream(side)
        if self.dpi.world > 1 and dist.get_backend(self.dpi.group) != "nccl":
            return None  # gloo collectives cannot be captured: eager replays
        graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(graph):
                self.outputs[k] = self._device_step(k)
        except Exception:  # noqa: BLE001  (a collective that refuses capture: run eagerly)
            torch.cuda.synchronize(self.dpi.device)
            self.capture_error = True
            return None
        return graph

    def step(self, k: int, host_in: dict, host_out: list):
        """Enqueue step k: host_in (pinned L, R, root, emit, tok) -> slot k % 2 ->
        host_out (pinned dL, dR, droot, d_emit, log_z)."""
        j = k % len(self.graphs)
        d = self.inputs[j]
        with torch.cuda.stream(self.s_in):
            if self.in_free[j] is not None:       # step k-2 has consumed these buffers
                self.s_in.wait_event(self.in_free[j])
            for key, t in host_in.items():
                d[key].copy_(t, non_blocking=True)
            self.in_ready[j].record(self.s_in)
        self.comp.wait_event(self.in_ready[j])
        if self.out_free[j] is not None:          # step k-2's results are on the host
            self.comp.wait_event(self.out_free[j])
        if self.graphs[j] is not None:
            self.graphs[j].replay()
        else:
            self.outputs[j] = self._device_step(j)
        self.in_free[j] = torch.cuda.Event()
        self.in_free[j].record(self.comp)
        self.out_ready[j].record(self.comp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.out_ready[j])
            for dst, src in zip(host_out, self.outputs[j]):
                dst.copy_(src, non_blocking=True)
            self.out_free[j] = torch.cuda.Event()
            self.out_free[j].record(self.s_out)

    def synchronize(self):
        self.s_out.synchronize()
        self.comp.synchronize()

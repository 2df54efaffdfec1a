"""Benchmark: inside fwd+bwd sentences/s at |N|=4096, length 40, batch 64
(BASELINE.json config 3) on 1..8 B200s, with the roofline of the dominant
kernel and the CPU oracle timed on the same host.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

(--gpus N > 1 without torchrun relaunches itself under torch.distributed.run.)
One step = forward + backward of the inside op over one batch of B sentences
per GPU (weak scaling, the default: B per rank; --scaling strong shards a
global B), through dp.DataParallelInside: the grammar gradients land in one
flat [dL | dR | droot] bucket that is all-reduced over NCCL when N > 1 (dL's
chunk overlapping dR's weight-gradient GEMM), the whole step captured as one
CUDA graph.  At N > 1 the other scaling mode is measured too
("scaling_other").  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {  # BASELINE.json configs (N = P = |N|)
    1: dict(n=64, batch=8, length=20),
    2: dict(n=1024, batch=32, length=30),
    3: dict(n=4096, batch=64, length=40),
    5: dict(n=8192, batch=128, length=40),
}
METRIC = "inside fwd+bwd sentences/sec @|N|=4096,len40 (1/2/4/8 B200) vs CPU; % roofline"
VOCAB = 64


# ---------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clock / throttle-reason sampling during the timed region.

    nvidia-smi polls every 20 ms with a host timestamp per line; only lines
    stamped inside [mark(), stop()] count (the default run's timed region is
    ~150 ms, so the sampler starts before it)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """Start of the timed region (lines read before it are dropped)."""
        self.t_mark = time.time()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        t_end = time.time()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t_mark = getattr(self, "t_mark", 0.0)
        for t_read, ln in self.lines:
            if not t_mark <= t_read <= t_end + 0.05:
                continue
            parts = [p.strip() for p in ln.split(",")][1:]  # drop the timestamp
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------- algorithmic work
def gather_launch_bytes(n: int, batch: int, length: int, m: int, gemm_esz: int,
                        chart_esz: int = 4) -> float:
    """Compulsory HBM bytes of the gather-backward launch for child width m.

    Child span (i, i+m) reads, per parent, a sibling row and the parent's LQ
    row.  Over one launch the left siblings b[w-m][i+m], the right siblings
    a[i-s][s] and the parents (every span wider than m) are each a bijection
    onto the S_m = (l-m)(l-m+1)/2 spans of width > m (resp. < l-m+1), and
    every parent row is shared by its left and right child, so the launch
    must read 2 * S_m distinct a/b rows (chart_esz bytes per element) and
    S_m outside-weight rows (fp32, or fp16 plus one fp32 exponent per 32
    columns with the fp16 chart); plus the child's own a, b rows (the -inf
    guard) and its 2N-wide G row written in the operand type."""
    l = length
    s_m = (l - m) * (l - m + 1) // 2
    n_m = l - m + 1
    lq_esz = 4.0 if chart_esz == 4 else 2.0 + 4.0 / 32
    return batch * (s_m * n * (2.0 * chart_esz + lq_esz)
                    + n_m * (2 * n * chart_esz + 2 * n * gemm_esz))


def split_launch_bytes(n: int, batch: int, length: int, w: int, gemm_esz: int,
                       chart_esz: int = 4) -> float:
    """Compulsory HBM bytes of the split-contraction launch for width w: every
    (span, split) pair reads the distinct rows a[m][i] and b[w-m][i+m]; the
    span's E row is written in the operand type (none at the top width)."""
    n_w = length - w + 1
    return batch * n_w * (2 * (w - 1) * n * chart_esz + (n * gemm_esz if w < length else 0))


def algorithmic_work(n: int, p: int, batch: int, length: int, gemm_esz: int, store_o: bool,
                     chart_esz: int = 4):
    """Per-class algorithmic flops / bytes of one fwd+bwd step.

    GEMM flops count only the live blocks: width 1 contracts over P, widths
    2..l-1 over N; dgrad and wgrad repeat the forward count.  Bandwidth-kernel
    bytes are the compulsory HBM bytes of each launch (split_launch_bytes,
    gather_launch_bytes): distinct chart rows read once per launch plus the
    rows written; re-reads across launches are counted, re-reads inside a
    launch are not."""
    l = length
    rows_w1 = batch * l
    rows_mid = batch * (l * (l - 1) // 2 - 1)          # widths 2..l-1
    f_fwd = 2.0 * rows_w1 * (2 * n) * p + 2.0 * rows_mid * (2 * n) * n
    spans_ge2 = batch * (l * (l - 1) // 2)             # widths 2..l
    split_bytes = (sum(split_launch_bytes(n, batch, l, w, gemm_esz, chart_esz)
                       for w in range(2, l + 1))
                   + spans_ge2 * n * (4.0 if store_o else 0))
    gather_bytes = sum(gather_launch_bytes(n, batch, l, m, gemm_esz, chart_esz)
                       for m in range(1, l))
    return {
        "gemm_fwd": ("tensor", f_fwd),
        "gemm_dgrad": ("tensor", f_fwd),
        "gemm_wgrad": ("tensor", f_fwd),
        "split_fwd": ("hbm", split_bytes),
        "gather_bwd": ("hbm", gather_bytes),
    }


def run_e2e(args, g, tokens, dpi, lengths, gvec, dev, batch, n, world, barrier):
    """End-to-end through host buffers, the reference-facing call pattern:
    every step copies its inputs (grammar tables + tokens) from pinned host
    memory to the GPU, runs fwd+bwd (+ the all-reduce at N > 1), and copies
    log_z and the GrammarGrad tables (dL, dR, droot, d_emit) back to pinned
    host memory.  Copies run on their own streams, double-buffered, so step
    k+1's H2D and step k's D2H overlap step k's compute -- what a training
    loop feeding the op does (dp.HostStreamedStep: the device part of a step
    is one CUDA-graph replay).  The timer covers all copies of all K steps
    (final sync included)."""
    import torch
    import torch.distributed as dist

    def pinned(a, dtype=torch.float32):
        return torch.as_tensor(np.array(a), dtype=dtype).pin_memory()

    # two distinct host input sets (as if each step brought new parameters)
    hosts = []
    for k in range(2):
        jitter = np.float32(1e-7 * k)
        hosts.append(dict(L=pinned(np.asarray(g.log_left) + jitter),
                          R=pinned(np.asarray(g.log_right) + jitter),
                          root=pinned(g.log_root), emit=pinned(g.log_emit),
                          tok=pinned(tokens, torch.int64)))
    outs = [[torch.empty(g.log_left.shape).pin_memory(), torch.empty(g.log_right.shape).pin_memory(),
             torch.empty(g.log_root.shape).pin_memory(),
             torch.empty(g.log_emit.shape).pin_memory(), torch.empty(batch).pin_memory()]
            for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in hosts[0].values())
    d2h = sum(t.numel() * t.element_size() for t in outs[0])
    from paper_2310_14997_b200.dp import HostStreamedStep
    hs = HostStreamedStep(dpi, VOCAB, lengths, gvec)   # one CUDA graph per buffer slot

    def run(nsteps):
        for k in range(nsteps):
            hs.step(k, hosts[k % 2], outs[k % 2])
        hs.synchronize()

    run(max(2, args.warmup))
    barrier()
    t0 = time.perf_counter()
    run(args.steps)
    barrier()
    ems = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([ems], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    return {"value": world * batch / (ems / 1e3), "unit": "sentences/s", "ms_per_step": ems,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "graphs": all(gr is not None for gr in hs.graphs),
            "path": "pinned host grammar+tokens -> H2D -> dp.HostStreamedStep: one CUDA-graph "
                    "replay of unary gather + engine fwd+bwd (C-ABI fi_inside_forward / "
                    "fi_inside_backward_ex, + all-reduce at N>1) + d_emit scatter -> D2H log_z + "
                    "GrammarGrad (dL, dR, droot, d_emit); copies on side streams, double-buffered "
                    "across steps; wall clock over K steps"}


def tensor_peak(gemm_dtype: str, peaks: dict) -> tuple[float, str]:
    """The tensor-core peak that matches the GEMM operand type.  Kernels here
    are timed over a sub-second region, so the burst (not the 4-s sustained)
    bf16 figure applies; tf32 uses the TF32 peak measured on the box
    (profiles/measured_tf32.json: torch.matmul tf32 8192^3, best of 10) when
    present, else half the bf16 burst (the dense tf32:bf16 ratio); fp32 mode
    issues three bf16 MMAs per product (hi*hi + hi*lo + lo*hi), so its
    algorithmic flops are held to a third of the bf16 burst."""
    if gemm_dtype == "tf32":
        f = ROOT / "profiles" / "measured_tf32.json"
        if f.exists():
            d = json.loads(f.read_text())
            return float(d["tf32_tflops"]), "measured tf32 burst (profiles/measured_tf32.json)"
        return peaks["bf16_tflops"] / 2, peaks["source"] + " bf16 burst / 2 (tf32 dense ratio)"
    if gemm_dtype == "fp32":
        return peaks["bf16_tflops"] / 3, peaks["source"] + " bf16 burst / 3 (bf16x3 operands)"
    return peaks["bf16_tflops"], peaks["source"] + " bf16 burst"


def roofline_block(prof: dict, steps: int, n: int, batch: int, length: int, esz: int,
                   chart_esz: int, gemm_dtype: str = "bf16") -> dict:
    """roofline{} of the dominant kernel class from per-class CUDA-event
    times (_lib.profile_collect over `steps` steps) and the algorithmic work."""
    peaks = measured_peaks()
    t_peak, t_src = tensor_peak(gemm_dtype, peaks)
    work = algorithmic_work(n, n, batch, length, esz, store_o=False, chart_esz=chart_esz)
    per_class = {}
    for name, (tot_ms, cnt) in prof.items():
        if cnt:
            per_class[name] = {"ms_per_step": tot_ms / steps, "launches_per_step": cnt // steps}
    dominant = max((k for k in per_class if k in work), key=lambda k: per_class[k]["ms_per_step"])
    bound, amount = work[dominant]
    k_ms = per_class[dominant]["ms_per_step"]
    if bound == "hbm":
        achieved = amount / (k_ms / 1e3) / 1e9
        peak = peaks["hbm_gbs"]
        unit = "GB/s"
    else:
        achieved = amount / (k_ms / 1e3) / 1e12
        peak = t_peak
        unit = "TFLOP/s"
    for name, d in per_class.items():
        if name in work:
            b, amt = work[name]
            d["achieved"] = amt / (d["ms_per_step"] / 1e3) / (1e9 if b == "hbm" else 1e12)
            d["unit"] = "GB/s" if b == "hbm" else "TFLOP/s"
            d["frac"] = d["achieved"] / (peaks["hbm_gbs"] if b == "hbm" else t_peak)
    # DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one launch
    # of the dominant class from the committed ncu --set full capture, next
    # to the compulsory bytes of that same launch (scripts/summarize_profiles.py)
    traffic, traffic_launch = None, None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic_launch = json.loads(tf.read_text()).get(dominant)
        if traffic_launch:
            traffic = traffic_launch.get("dram_bytes")
    return {"kernel": dominant, "bound": bound, "achieved": achieved, "peak": peak,
            "unit": unit, "frac": achieved / peak, "traffic": traffic,
            "traffic_launch": traffic_launch,
            "method": "algorithmic work per step / CUDA-event time of the class's launches "
                      "(same K steps re-run with per-launch events)",
            "peak_source": t_src if bound == "tensor" else peaks["source"] + " HBM copy",
            "tensor_peak": {"value": t_peak, "source": t_src},
            "per_class": per_class}


def init_dist(world: int, local: int):
    """One process per GPU over NCCL (FI_DIST_BACKEND=gloo with ranks sharing
    devices exercises the multi-rank code path on a single-GPU box)."""
    import torch
    import torch.distributed as dist
    ngpu = max(torch.cuda.device_count(), 1)
    # more ranks than GPUs (a multi-rank dry run on a 1-GPU box): NCCL refuses
    # two ranks on one device, so those runs use gloo (eager, no graphs)
    backend = os.environ.get("FI_DIST_BACKEND", "nccl" if world <= ngpu else "gloo")
    if world > 1 and backend == "nccl":
        # NCCL's communicator init lines (one per rank) stay in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dev_idx = local % ngpu
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev, backend


# -------------------------------------------------------------- our arm
def timed_steps(step, steps, warmup, use_graph, barrier, lib, dev):
    """W eager warm-up steps, then (optionally) capture one step as a CUDA
    graph -- NCCL all-reduce included when N > 1 -- and time K steps with
    CUDA events between barriers.  Returns (ms per step, our kernel launches
    in the timed region, launch mode)."""
    import torch
    for _ in range(warmup):
        step()
    barrier()
    graph, graph_launches, mode = None, 0, "eager"
    if use_graph:
        try:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                for _ in range(2):
                    step()
            torch.cuda.current_stream(dev).wait_stream(side)
            barrier()
            graph = torch.cuda.CUDAGraph()
            c0 = lib.fi_launch_count()
            with torch.cuda.graph(graph):
                step()
            graph_launches = int(lib.fi_launch_count() - c0)
            for _ in range(2):
                graph.replay()
            barrier()
            mode = "cuda-graph replay"
        except Exception as e:  # noqa: BLE001  (reported in the JSON line)
            graph = None
            mode = f"eager (graph capture failed: {type(e).__name__}: {str(e)[:120]})"
            torch.cuda.synchronize(dev)
            barrier()
    launch0 = lib.fi_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1) / steps
    launches = graph_launches * steps if graph is not None else int(lib.fi_launch_count() - launch0)
    if graph is not None:
        del graph
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
    return ms, launches, mode


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2310_14997_b200 import _lib
    from paper_2310_14997_b200.dp import DataParallelInside
    from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
    from paper_2310_14997_b200.ops import check_lengths

    dev, backend = init_dist(world, local)
    cfg = CONFIGS[args.config]
    n, length = cfg["n"], args.length or cfg["length"]
    batch_cfg = args.batch or cfg["batch"]

    def per_gpu(scaling):
        if scaling == "strong":
            if batch_cfg % world:
                raise SystemExit(f"strong scaling needs batch % gpus == 0 ({batch_cfg} % {world})")
            return batch_cfg // world
        return batch_cfg

    batch = per_gpu(args.scaling)
    g = random_grammar(GrammarDims(n, n, VOCAB), seed=0)
    L = torch.tensor(g.log_left, dtype=torch.float32, device=dev)
    R = torch.tensor(g.log_right, dtype=torch.float32, device=dev)
    root = torch.tensor(g.log_root, dtype=torch.float32, device=dev)
    emit = torch.tensor(g.log_emit, dtype=torch.float32, device=dev)
    lib = _lib.load()
    chart_fmt = int(_lib.chart_layout(_lib.shape(n, n, batch, length, args.gemm_dtype, False,
                                                 args.chart_dtype)).chart_fmt)
    use_graph = args.graph != 0 and backend != "gloo"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def make(bsz):
        """This rank's shard: tokens default_rng(1 + rank), lengths, the
        data-parallel engine and the step closure (the loss is the global
        mean NLL: grad_log_z = -1 / global batch, train.py:218)."""
        tokens = np.random.default_rng(1 + rank).integers(0, VOCAB, size=(bsz, length))
        tok_d = torch.as_tensor(tokens, device=dev)
        unary = emit.t()[tok_d].contiguous()
        lengths = torch.full((bsz,), length, dtype=torch.int32, device=dev)
        check_lengths(lengths, length)  # once: the timed steps skip the host read
        gvec = torch.full((bsz,), -1.0 / (bsz * world), device=dev)
        dpi = DataParallelInside(n, n, bsz, length, args.gemm_dtype, args.chart_dtype, dev,
                                 slots=2)
        return tokens, unary, lengths, gvec, dpi

    tokens, unary, lengths, gvec, dpi = make(batch)

    def step():
        return dpi.step(L, R, root, unary, lengths, gvec)

    # ---- device-resident timed region (the clock sampler runs from the
    # warm-up on; only its samples inside the timed region count)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.mark()
    ms, gpu_launches, launch_mode = timed_steps(step, args.steps, args.warmup, use_graph, barrier,
                                                lib, dev)
    clk = clocks.stop()
    log_z = dpi.log_z
    loss_val = float(-(log_z.sum()) / batch)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-kernel-class CUDA-event timing: the same K steps again with events
    # bracketing every library launch on its stream (kept out of the headline
    # region above so the events cannot perturb it)
    _lib.profile_enable(True)
    barrier()
    for _ in range(args.steps):
        step()
    barrier()
    _lib.profile_enable(False)
    prof = _lib.profile_collect()
    value = world * batch / (ms / 1e3)

    # ---- the other scaling mode at N > 1 (weak: B per GPU; strong: B global)
    other = None
    if world > 1 and not args.no_other_scaling:
        mode2 = "strong" if args.scaling == "weak" else "weak"
        b2 = per_gpu(mode2)
        del dpi
        torch.cuda.empty_cache()
        _, unary2, lengths2, gvec2, dpi2 = make(b2)
        ms2, _, lm2 = timed_steps(lambda: dpi2.step(L, R, root, unary2, lengths2, gvec2),
                                  args.steps, args.warmup, use_graph, barrier, lib, dev)
        t = torch.tensor([ms2], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms2 = float(t.item())
        other = {"scaling": mode2, "batch_per_gpu": b2, "global_batch": b2 * world,
                 "ms_per_step": ms2, "value": world * b2 / (ms2 / 1e3), "unit": "sentences/s",
                 "launch": lm2}
        del dpi2
        torch.cuda.empty_cache()
        tokens, unary, lengths, gvec, dpi = make(batch)

    # ---- end-to-end through host buffers (reference-facing call pattern)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, g, tokens, dpi, lengths, gvec, dev, batch, n, world, barrier)

    # ---- roofline of the dominant kernel class
    esz = 4 if args.gemm_dtype == "tf32" else 2
    chart_esz = 2 if chart_fmt == _lib.FI_CHART_F16 else 4
    roofline = roofline_block(prof, args.steps, n, batch, length, esz, chart_esz,
                              args.gemm_dtype)

    # ---- CPU baseline (oracle port) on rank 0, N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(g, tokens[:1], length)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": ("fp16 linear a/b chart (fp32 o, lq, accumulators)" if chart_esz == 2
                      else "fp32 chart") + ", "
                     + {"bf16": "bf16", "tf32": "tf32",
                        "fp32": "bf16x3 (fp32-accurate)"}[args.gemm_dtype]
                     + " GEMM operands, fp32 accumulate",
            "data": "synthetic: random_grammar(GrammarDims(N,N,64), seed=0) Dirichlet(1) rows; "
                    "uniform tokens default_rng(1+rank)",
            "config": {"workload": f"config {args.config}: SimplePCFG |N|={n} (N=P={n}), "
                                   f"length {length}, batch {batch} per GPU, fwd+bwd",
                       "n_nt": n, "n_pt": n, "length": length, "batch_per_gpu": batch,
                       "global_batch": batch * world, "gemm_dtype": args.gemm_dtype,
                       "chart_dtype": "fp16" if chart_esz == 2 else "fp32",
                       "launch": launch_mode, "dist_backend": backend if world > 1 else None,
                       "parallelism": f"dp{world}",
                       "collective": ("one flat [dL|dR|droot] bucket, all-reduced in 2 chunks "
                                      "(dL overlapping dR's wgrad GEMM)") if world > 1 else None,
                       "l2": "working set ~4 GB chart per step >> 126 MB L2 (no flush needed)"},
            "scaling_other": other,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "loss": loss_val,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------ training workload
TRAIN_METRIC = "neural SimplePCFG train step sentences/sec @|N|=4096,len40,d=512"


def run_train(args, world, rank, local):
    """--workload train: the full training step of train.py:201-227 on the GPU
    (neural parameterisation d=512 -> inside fwd+bwd on the engine ->
    autograd -> one all-reduce of the parameter gradients -> clip -> Adam),
    B sentences per GPU (weak scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2310_14997_b200 import _lib, neural
    from paper_2310_14997_b200.grammar import GrammarDims

    dev, _ = init_dist(world, local)
    cfg = CONFIGS[args.config]
    n, length = cfg["n"], args.length or cfg["length"]
    batch = args.batch or cfg["batch"]
    dims = GrammarDims(n, n, VOCAB)
    ts = neural.TrainStep(neural.init_params(dims, 512, 0, device=dev),
                          neural.TrainConfig(gemm_dtype=args.gemm_dtype))
    tok = torch.as_tensor(np.random.default_rng(1 + rank).integers(0, VOCAB, (batch, length)),
                          device=dev)
    lengths = torch.full((batch,), length, dtype=torch.int32, device=dev)
    lib = _lib.load()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        ts.step(tok, lengths, global_batch=batch * world)
    barrier()
    launch0 = lib.fi_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark()
    e0.record()
    for _ in range(args.steps):
        loss = ts.step(tok, lengths, global_batch=batch * world)
    e1.record()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    gpu_launches = int(lib.fi_launch_count() - launch0)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    _lib.profile_enable(True)
    for _ in range(args.steps):
        ts.step(tok, lengths, global_batch=batch * world)
    barrier()
    _lib.profile_enable(False)
    prof = _lib.profile_collect()
    chart_fmt = int(_lib.chart_layout(_lib.shape(n, n, batch, length, args.gemm_dtype)).chart_fmt)
    roofline = roofline_block(prof, args.steps, n, batch, length,
                              4 if args.gemm_dtype == "tf32" else 2,
                              2 if chart_fmt == _lib.FI_CHART_F16 else 4)
    inside_ms = sum(d["ms_per_step"] for k, d in roofline["per_class"].items() if k != "param")
    param_ms = roofline["per_class"].get("param", {}).get("ms_per_step", 0.0)
    if rank == 0:
        print(json.dumps({
            "metric": TRAIN_METRIC, "value": world * batch / (ms / 1e3), "unit": "sentences/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": f"{args.gemm_dtype} GEMM operands, fp32 parameters / Adam",
            "data": "synthetic uniform tokens; init_params(seed=0)",
            "config": {"workload": f"config {args.config} train step: neural PCFG N=P={n}, d=512, "
                                   f"length {length}, batch {batch} per GPU",
                       "parallelism": f"dp{world}", "global_batch": batch * world},
            "clocks": clk, "gpu_launches": gpu_launches, "loss": float(loss),
            "inside_engine_ms_per_step": inside_ms,
            "score_tables_ms_per_step": param_ms,
            "mlp_and_optimizer_ms_per_step": ms - inside_ms - param_ms,
            "roofline": roofline}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline_sample(g, tokens, length):
    """Time the CPU oracle (float64 NumPy port of the reference path) on a
    bounded sample: one sentence of the workload, forward + backward."""
    from oracle import flashinside_oracle as O
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(_cpu_threads())
    except ImportError:
        pass
    un = O.unary_from_tokens(np.asarray(g.log_emit), tokens, length)
    t0 = time.perf_counter()
    O.inside_batch(g.log_left, g.log_right, g.log_root, un, np.array([length]))
    dt = time.perf_counter() - t0
    return {"value": tokens.shape[0] / dt, "unit": "sentences/s", "cores": _cpu_threads(),
            "kind": "port", "seconds": dt,
            "sample": f"{tokens.shape[0]} sentence (l={length}) of the workload, fwd + "
                      "GEMM-form bwd, float64 NumPy/OpenBLAS, all host threads"}


# --------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """The reference's CPU path (oracle port: the reference is Python and does
    not travel to the GPU box) on this host's cores, rank 0 only."""
    if rank != 0:
        return
    from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
    from oracle import flashinside_oracle as O
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(_cpu_threads())
    except ImportError:
        pass
    cfg = CONFIGS[args.config]
    n, length = cfg["n"], args.length or cfg["length"]
    g = random_grammar(GrammarDims(n, n, VOCAB), seed=0)
    rng = np.random.default_rng(1)
    sample = 1  # sentences per step: a bounded sample of the batch
    tok = rng.integers(0, VOCAB, size=(args.steps + args.warmup, length))
    un_all = O.unary_from_tokens(np.asarray(g.log_emit), tok, length)
    for k in range(args.warmup):
        O.inside_batch(g.log_left, g.log_right, g.log_root, un_all[k:k + 1], np.array([length]))
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        O.inside_batch(g.log_left, g.log_right, g.log_root, un_all[k:k + 1], np.array([length]))
    dt = (time.perf_counter() - t0) / args.steps
    value = sample / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sentences/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (same grammar/tokens generator as our arm)",
        "config": {"workload": f"config {args.config}: SimplePCFG |N|={n}, length {length}, "
                               f"{sample} sentence per step (bounded sample), fwd+bwd",
                   "n_nt": n, "length": length, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "sentences/s", "cores": _cpu_threads(),
                         "kind": "port",
                         "sample": f"{sample} sentence per step; float64 NumPy port of "
                                   "inside_flash + inside_backward (GEMM form)"},
        "e2e": {"value": value, "unit": "sentences/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(nproc: int, argv: list) -> int:
    """Run this script under torch.distributed.run with `nproc` ranks on this
    node (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *argv]
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["inside", "train"], default="inside",
                    help="inside: the op's fwd+bwd (headline); train: the full GPU training step")
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), default=3)
    ap.add_argument("--length", type=int, default=None,
                    help="sentence length override (config 4: the 10..60 sweep at |N|=4096)")
    ap.add_argument("--batch", type=int, default=None, help="sentences per GPU (weak) / "
                    "global (strong); default: the config's batch")
    ap.add_argument("--gemm-dtype", choices=["bf16", "tf32", "fp32"], default="bf16")
    ap.add_argument("--chart-dtype", choices=["auto", "fp32", "fp16"], default="auto")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--graph", type=int, default=-1,
                    help="1: time CUDA-graph replays of the captured step; 0: eager launches; "
                         "-1 (default): graphs on one GPU, eager under torchrun")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-scaling", action="store_true",
                    help="N > 1: skip the second measurement in the other scaling mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: launch N ranks of this same command
        return relaunch(args.gpus, sys.argv[1:] if argv is None else list(argv))
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.workload == "train":
        run_train(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()

"""Summarise ncu outputs (launch list CSV + --set full reports) into profiles/.

    python scripts/summarize_profiles.py --tag r01 --launches gpurun_out/launches.csv \
        --reps gpurun_out/prof_*.ncu-rep

Writes profiles/<tag>_launches_summary.md, profiles/<tag>_ncu_kernels.json and
profiles/ncu_traffic.json (per kernel class: DRAM bytes of the captured
launch and its algorithmic bytes, read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "second": 1e3, "s": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
         "GB": 1e9}


def short(name: str) -> str:
    return re.sub(r"\(.*", "", name).replace("void fi::", "").replace("void ", "")


def launches(path: Path, tag: str) -> str:
    rows = list(csv.reader(path.read_text().splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ks = [(r[ki], float(r[vi].replace(",", "")) * SCALE[r[ui]]) for r in data if len(r) > vi]
    step = ks[len(ks) // 2:]  # second of two identical steps (first is warm-up)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, ms in step:
        agg[short(name)][0] += 1
        agg[short(name)][1] += ms
    tot = sum(ms for _, ms in step)
    out = [f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none)",
           "", "Second of two identical fwd+bwd steps; ncu serialises and cold-starts every",
           "launch, so compare the SHARES with bench.py's per-class CUDA-event times.",
           f"Total {tot:.2f} ms over {len(step)} launches.", "",
           "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k[:90]}` | {c} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    return "\n".join(out) + "\n"


WANT = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "regs": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}


def report(path: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"file": path.name, "kernel": short(r[hdr.index("Kernel Name")]),
             "grid": r[hdr.index("Grid Size")], "block": r[hdr.index("Block Size")]}
        for key, metric in WANT.items():
            if metric not in hdr:
                continue
            j = hdr.index(metric)
            try:
                v = float(r[j].replace(",", ""))
            except ValueError:
                continue
            u = units[j]
            if key == "time_ms":
                v *= SCALE.get(u, 1.0)
            elif key.startswith("dram_") and key != "dram_pct_peak":
                v *= BYTES.get(u, 1.0)
            d[key] = v
        res.append(d)
    return res


def classify(k: dict) -> str | None:
    name = k["kernel"]
    if "split_fwd" in name:
        return "split_fwd"
    if "gather_bwd" in name:
        return "gather_bwd"
    m = re.match(r"k_gemm<[^,]+, \d+, \d, \d, (\d)", name)
    if m:
        return {"0": "gemm_fwd", "5": "gemm_fwd", "1": "gemm_dgrad", "6": "gemm_dgrad",
                "2": "gemm_dgrad", "3": "gemm_wgrad"}.get(m.group(1))
    return None


def traffic(kernels: list[dict], n: int, batch: int, length: int, esz: int,
            chart_esz: int, widths: dict) -> dict:
    """Per kernel class: DRAM bytes of the captured launch next to the
    compulsory (algorithmic) bytes of that same launch (bench.py formulas)."""
    import sys
    sys.path.insert(0, str(ROOT))
    import bench
    out = {}
    for k in kernels:
        cls = classify(k)
        if cls is None or "dram_read" not in k:
            continue
        gy = int(k["grid"].strip("()").split(",")[1])
        d = {"dram_bytes": k["dram_read"] + k["dram_write"], "time_ms": k["time_ms"],
             "launch": f"{k['file']} grid {k['grid']}"}
        if cls in ("split_fwd", "gather_bwd"):
            # the captured launch's width (persistent grids do not encode it)
            width = widths.get(cls) or length - gy // batch + 1
            fn = bench.split_launch_bytes if cls == "split_fwd" else bench.gather_launch_bytes
            d["width"] = width
            d["algorithmic_bytes"] = fn(n, batch, length, width, esz, chart_esz)
            d["dram_over_algorithmic"] = d["dram_bytes"] / d["algorithmic_bytes"]
            d["achieved_gbs_under_ncu"] = d["algorithmic_bytes"] / (k["time_ms"] * 1e-3) / 1e9
        if cls in ("gemm_fwd", "gemm_dgrad") and widths.get("gemm"):
            # the captured launch's width: M = batch * (l - w + 1) rows, K x N = N x 2N
            w = widths["gemm"]
            flops = 2.0 * batch * (length - w + 1) * (2 * n) * n
            d["width"] = w
            d["algorithmic_tflop"] = flops / 1e12
            d["achieved_tflops_under_ncu"] = flops / (k["time_ms"] * 1e-3) / 1e12
        out[cls] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--length", type=int, default=40)
    ap.add_argument("--esz", type=int, default=2, help="GEMM operand bytes (bf16 2, tf32 4)")
    ap.add_argument("--chart-esz", type=int, default=2, help="a/b chart bytes (fp16 2, fp32 4)")
    ap.add_argument("--split-width", type=int, default=20, help="width of the captured split launch")
    ap.add_argument("--gather-width", type=int, default=20, help="child width of the captured gather")
    ap.add_argument("--gemm-width", type=int, default=0, help="width of the captured fwd / dgrad GEMM launches")
    ap.add_argument("--launches")
    ap.add_argument("--reps", nargs="*", default=[])
    args = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    if args.launches:
        text = launches(Path(args.launches), args.tag)
        (prof / f"{args.tag}_launches_summary.md").write_text(text)
        print(text)
    kernels = []
    for rp in args.reps:
        kernels += report(Path(rp))
    if kernels:
        (prof / f"{args.tag}_ncu_kernels.json").write_text(json.dumps(kernels, indent=1))
        for k in kernels:
            print(json.dumps(k))
        tr = traffic(kernels, args.n, args.batch, args.length, args.esz, args.chart_esz,
                     {"split_fwd": args.split_width, "gather_bwd": args.gather_width,
                      "gemm": args.gemm_width})
        (prof / "ncu_traffic.json").write_text(json.dumps(tr, indent=1))
        print(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main()

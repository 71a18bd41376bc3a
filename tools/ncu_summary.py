"""Summarise ncu reports / launch lists into profiles/ (committed evidence).

    python tools/ncu_summary.py gpurun_out/prof_render2.ncu-rep > profiles/r1_render.txt
    python tools/ncu_summary.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>16s} {units[i]}")
        stalls = [(int(float(r[i])), hdr[i][len(STALLS):]) for i in range(len(hdr))
                  if hdr[i].startswith(STALLS) and not hdr[i].endswith("not_issued") and r[i] not in ("", "n/a")]
        tot = sum(s for s, _ in stalls) or 1
        print("  warp stall samples (top):")
        for s, n in sorted(stalls, reverse=True)[:8]:
            print(f"    {n:40s} {s:8d} {100.0 * s / tot:5.1f}%")


def hot_lines(path, top=30):
    """Top CUDA source lines by warp-stall samples (needs -lineinfo + --import-source)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if "# Samples" in r)
    si, ie = hdr.index("# Samples"), hdr.index("Instructions Executed")
    res = []
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) > si and r[2] == "-":
            try:
                res.append((int(r[si]), int(r[0]), int(r[ie] or 0), r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in res) or 1
    print(f"  hot source lines (of {tot} samples):")
    for n, line, inst, src in sorted(res, reverse=True)[:top]:
        print(f"    {100.0 * n / tot:5.1f}%  L{line:<5d} inst {inst:>11d}  {src}")


def launches(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    agg = {}
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        agg.setdefault(k, []).append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"launches: {len(rows)}  total {tot / 1e6:.3f} ms (ncu serialised, cold cache)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:40s} n={len(v):4d} mean {sum(v) / len(v) / 1e3:9.1f} us  share {100 * sum(v) / tot:5.1f}%")


def kernel_json(path):
    """Per-kernel mean time and DRAM bytes per launch (read by bench.py as roofline.traffic)."""
    import json

    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    agg = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("rsim::", "")
        v = lambda k: float(r[hdr.index(k)])  # noqa: E731
        a = agg.setdefault(name, {"launches": 0, "gpu_time_ms": 0.0, "dram_bytes": 0.0, "inst": 0.0,
                                  "grid": int(v("launch__grid_size"))})
        a["launches"] += 1
        a["inst"] += v("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in hdr else 0.0
        a["gpu_time_ms"] += v("gpu__time_duration.sum")
        a["dram_bytes"] += (v("dram__bytes_read.sum") + v("dram__bytes_write.sum")) * 1e6
    out = {k: {"launches": a["launches"], "grid": a["grid"], "gpu_time_ms": a["gpu_time_ms"] / a["launches"],
               "dram_bytes_per_launch": a["dram_bytes"] / a["launches"],
               "warp_inst_per_launch": a["inst"] / a["launches"]} for k, a in agg.items()}
    print(json.dumps({"source": path.split("/")[-1], "kernels": out}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--json":
        kernel_json(sys.argv[2])
    elif sys.argv[1] == "--lines":
        report(sys.argv[2])
        hot_lines(sys.argv[2])
    else:
        report(sys.argv[1])

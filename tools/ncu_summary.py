"""Summarise ncu outputs into profiles/ (run here, on the CPU box, after gpurun brought them back).

usage: python tools/ncu_summary.py <report.ncu-rep> <out.json> [launches.csv]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "gpc__cycles_elapsed.max", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",   # tcgen05 (UTC) tensor pipe busy
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in KEYS or h in ("Kernel Name", "ID"):
                d[h] = r[i] + (f" {units[i]}" if units[i] and h in KEYS else "")
        kernels.append(d)
    return kernels


def details(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "details"], capture_output=True, text=True).stdout
    keep = [l.rstrip() for l in out.splitlines()
            if any(k in l for k in ("Throughput", "highest-utilized", "TC is", "Duration", "Elapsed Cycles",
                                    "SM Frequency", "DRAM Frequency", "Registers Per", "Cluster", "Achieved"))]
    return keep


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[i + 1:]:
        name = r[ki].split("(")[0][:90]
        v = float(r[vi].replace(",", ""))
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    total = sum(t for _, t in agg.values())
    return {k: {"launches": n, "total_us": round(t / 1e3, 1), "share": round(t / total, 4)}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    doc = {"report": rep, "kernels": raw(rep), "details": details(rep)}
    if len(sys.argv) > 3:
        doc["launch_list"] = launches(sys.argv[3])
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc["kernels"], indent=1))

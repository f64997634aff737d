"""Turn the round's op-kernel ncu captures into the bench's per-shape traffic files and summaries.

For every gpurun_out/r2_ncu_op_<key>_g<G>_<kind>_<agent>.ncu-rep (tools/_r2_evidence.sh) writes
  profiles/r02_ncu_traffic_<key>_g<G>_<kind>_<agent>.json  {"dram_bytes_per_launch": read + write, ...}
  profiles/r02_ncu_op_<key>_g<G>_<kind>_<agent>.json       (tools/ncu_summary.py summary of the capture)
bench.traffic_for() reads the first one as roofline.traffic for exactly that (workload, G, schedule, agent).
usage: python tools/traffic_files.py [gpurun_out]
"""
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402


def bytes_of(v: str) -> float:
    num, unit = v.split()[0], (v.split()[1] if len(v.split()) > 1 else "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(num.replace(",", "")) * scale


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    for rep in sorted(glob.glob(os.path.join(src, "r2_ncu_op_*.ncu-rep"))):
        m = re.match(r"r2_ncu_op_(\w+?)_g(\d+)_(\w+)_(dma|core)\.ncu-rep", os.path.basename(rep))
        if not m:
            continue
        key, G, kind, agent = m.groups()
        kern = ncu_summary.raw(rep)
        if not kern:
            print("empty", rep)
            continue
        k0 = kern[0]
        rd, wr = bytes_of(k0["dram__bytes_read.sum"]), bytes_of(k0["dram__bytes_write.sum"])
        tag = f"{key}_g{G}_{kind}_{agent}"
        with open(os.path.join(ROOT, "profiles", f"r02_ncu_traffic_{tag}.json"), "w") as f:
            json.dump({"config": key, "ranks": int(G), "schedule": kind, "comm_agent": agent,
                       "kernel": k0["Kernel Name"], "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                       "dram_write": wr, "ncu_duration": k0["gpu__time_duration.sum"],
                       "source": f"ncu --set full --clock-control none, 1 launch of the op's tile kernel "
                                 f"(tools/op_once.py {key} {kind} {agent} 3 {G}); copies complete before the "
                                 f"kernel under the profiler"}, f, indent=1)
        with open(os.path.join(ROOT, "profiles", f"r02_ncu_op_{tag}.json"), "w") as f:
            json.dump({"report": os.path.relpath(rep, ROOT), "kernels": kern,
                       "details": ncu_summary.details(rep)}, f, indent=1)
        print(tag, round((rd + wr) / 1e9, 3), "GB", k0["gpu__time_duration.sum"])


if __name__ == "__main__":
    main()

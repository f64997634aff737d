"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) into JSON.

usage: python tools/launch_summary.py gpurun_out/launches_c2.csv profiles/r01_launches_c2.json "<command>"

Per kernel name: launches, mean/min/max duration (µs, cold-cache, serialised by
ncu). ``ficco_share`` is the tile kernel's share of all non-torch-housekeeping
kernel time (the L2-flush fill and input-generation kernels excluded).
"""
import collections
import csv
import json
import statistics
import sys

HOUSEKEEPING = ("FillFunctor", "distribution_", "CatArrayBatchedCopy", "bfloat16_copy_kernel", "AUnaryFunctor",
                "BUnaryFunctor", "CUDAFunctorOnSelf_add", "AbsFunctor", "BinaryFunctor", "reduce_kernel",
                "CompareFunctor", "CUDAFunctor_add", "direct_copy_kernel", "simt_sgemm")


def main(src: str, dst: str, command: str) -> None:
    rows = [r for r in csv.DictReader(line for line in open(src) if line.startswith('"'))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    per = collections.defaultdict(list)
    for r in rows:
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}[r["Metric Unit"]]
        per[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) * scale)
    kernels = []
    for name, ts in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        kernels.append({"kernel": name, "launches": len(ts), "total_us": round(sum(ts), 1),
                        "mean_us": round(statistics.mean(ts), 2), "min_us": round(min(ts), 2),
                        "max_us": round(max(ts), 2),
                        "housekeeping": any(h in name for h in HOUSEKEEPING)})
    work = [k for k in kernels if not k["housekeeping"]]
    total = sum(k["total_us"] for k in work)
    tile = sum(k["total_us"] for k in work if "tile_gemm_kernel" in k["kernel"])
    out = {"command": command, "source": src, "launches": len(rows),
           "ficco_share": round(tile / total, 4) if total else None,
           "note": "ncu serialises kernels: FiCCO copy programs run before the tile kernel under the profiler "
                   "(FICCO_SERIALIZE auto-on), so per-launch times are cold-cache and flag-wait-free",
           "kernels": kernels}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("launches", "ficco_share")}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")

"""Measured vs simulated timelines in the reference's trace schema.

C2 (Llama-3-8B MLP up-proj AG->GEMM, (M, N, K) = (8192, 3584, 4096), G = 8, rank 0, virtual
peers): for every executable schedule, ``executor.execute`` (the measured twin of
``simulate``) and ``simulate`` with the B200 machine file and calibration
(data/machine_b200.json, data/calibration_b200.json) each give a ``SimResult``; both are written
with ``export_trace_csv`` (engine.py:310-318) so they diff column for column, plus a JSON
summary of the makespans. Usage: python tools/trace_compare.py [out_dir]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_10236_b200 import executor, machines, ops, runtime  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind, build_plan  # noqa: E402
from paper_2512_10236_b200.simulator import export_trace_csv, simulate  # noqa: E402

KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
         "uniform_fused_2d"]


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    os.makedirs(out_dir, exist_ok=True)
    runtime.load_library()
    G, R, K, N = 8, 1024, 4096, 3584
    spec = machines.b200_machine()
    model = machines.b200_calibration()
    gen = torch.Generator(device="cuda").manual_seed(0)
    shards = [(torch.rand(R, K, generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(G)]
    w = (torch.randn(N, K, generator=gen, device="cuda") / K ** 0.5).to(torch.bfloat16)
    grp = ops.FiccoGroup.virtual_group(G, 0)
    summary = {}
    try:
        for kind in KINDS:
            sc = ops._scenario("c2_ag_gemm", G * R, N, K, G)
            plan = build_plan(sc, ScheduleKind(kind))
            _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
            grp.load_peer_shards(low, shards)
            _, measured = executor.execute(plan, shards[0], w, grp)
            simulated = simulate(plan, spec.machine, spec.topo, model)
            for tag, res in (("measured", measured), ("simulated", simulated)):
                with open(os.path.join(out_dir, f"trace_c2_{kind}_{tag}.csv"), "w") as f:
                    f.write(export_trace_csv(res))
            mine = [s for s in simulated.timeline if s.gpu == 0]
            summary[kind] = {"measured_makespan_us": round(measured.makespan * 1e6, 2),
                             "simulated_makespan_us": round(simulated.makespan * 1e6, 2),
                             "measured_spans": len(measured.timeline), "simulated_spans_rank0": len(mine)}
            print(kind, summary[kind], flush=True)
    finally:
        grp.close()
    with open(os.path.join(out_dir, "trace_c2_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()

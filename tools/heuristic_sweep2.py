"""C5 (BASELINE.json configs[4]): the schedule heuristic vs the MEASURED exhaustive best, and the B200 t_ref fit.

Per scenario (the BASELINE configs that fit one GPU + every corpus / synthetic-grid shape whose per-GPU GEMM
runs in well under a second): every executable kind (serial, shard ring, the four fine-grain kinds) as the
public op on a virtual 8-rank group, timed INTERLEAVED step by step (same clocks for all kinds), L2 flushed
before each call, 3 rounds x 7 steps, median. ``selector.validate_heuristic`` (heuristic.py:74-115) is then
scored with these measured makespans (makespan_fn) for a grid of t_ref values and the reference default
t_ref = 1 s; the fit keeps the t_ref with the most agreements (ties: least mean regret, then closest to 1 s).
usage: python tools/heuristic_sweep2.py [out_dir]   -> <out>/heuristic_sweep2.json
"""
import json
import math
import os
import statistics
import sys
from importlib import resources

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_10236_b200 import machines, ops, runtime, selector  # noqa: E402
from paper_2512_10236_b200.cli_data import synthetic_grid  # noqa: E402
from paper_2512_10236_b200.domain import parse_scenarios  # noqa: E402
from paper_2512_10236_b200.routing import PlanError, ScheduleKind, supported_kinds  # noqa: E402

MAX_FLOPS = 1.2e14
MAX_BYTES = 40e9
KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
         "uniform_fused_2d"]


def fits(sc) -> bool:
    g = sc.gemm
    return 2 * g.m * g.n * g.k <= MAX_FLOPS and 2 * (2 * g.m * g.k + g.m * g.n) <= MAX_BYTES


def measure(sc, flush, rounds=3, steps=7):
    G, M, N, K = sc.n_gpus, sc.gemm.m, sc.gemm.n, sc.gemm.k
    R = M // G
    gen = torch.Generator(device="cuda").manual_seed(0)
    shards = [(torch.rand(R, K, generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(G)]
    w = (torch.randn(N, K, generator=gen, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    grp = ops.FiccoGroup.virtual_group(G, 0)
    fns, names = [], []
    try:
        for kind in KINDS:
            try:
                _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
            except PlanError:
                continue
            grp.load_peer_shards(low, shards)
            fns.append(lambda kd=kind: ops.all_gather_matmul(shards[0], w, kind=kd, group=grp, out=out))
            names.append(kind)
        for fn in fns * 2:
            fn()
        torch.cuda.synchronize()
        samples = {n: [] for n in names}
        for _ in range(rounds):
            evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(steps)] for _ in fns]
            for i in range(steps):
                for fn, ev in zip(fns, evs):
                    flush()
                    ev[i][0].record()
                    fn()
                    ev[i][1].record()
            torch.cuda.synchronize()
            for n, ev in zip(names, evs):
                samples[n].append(statistics.median(a.elapsed_time(b) for a, b in ev))
        grp.comm.check()
    finally:
        grp.close()
    return {n: statistics.median(v) * 1e-3 for n, v in samples.items()}  # seconds


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    os.makedirs(out_dir, exist_ok=True)
    runtime.load_library()
    spec = machines.b200_machine()
    model = machines.b200_calibration()
    scen = [ops._scenario("C2_llama3_8b_up", 8192, 3584, 4096, 8), ops._scenario("C1_bf16", 4096, 4096, 4096, 8),
            ops._scenario("C3p_llama3_70b_up", 16384, 7168, 8192, 8),
            ops._scenario("C4_cp_qk_T", 131072, 16384, 128, 8)]
    corpus = parse_scenarios(resources.files("paper_2512_10236_b200.data").joinpath("scenarios_corpus.csv")
                             .read_text())
    scen += [s for s in list(corpus) + list(synthetic_grid()) if fits(s)]
    only = os.environ.get("SWEEP_ONLY")
    if only:
        scen = [s for s in scen if s.name in only.split(",")]
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    cache = {}
    table = []
    for sc in scen:
        t = measure(sc, flush)
        g = sc.gemm
        for kind, secs in t.items():
            cache[(g.m, g.n, g.k, sc.n_gpus, ScheduleKind(kind))] = secs
        fine = {k: v for k, v in t.items() if k in ("uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
                                                     "uniform_fused_2d")}
        row = {"scenario": sc.name, "m": g.m, "n": g.n, "k": g.k, "flops": 2 * g.m * g.n * g.k,
               "us": {k: round(v * 1e6, 2) for k, v in t.items()},
               "best_fine": min(fine, key=fine.get)}
        table.append(row)
        print(row, flush=True)

    def makespan(plan):
        g = plan.scenario.gemm
        return cache.get((g.m, g.n, g.k, plan.scenario.n_gpus, plan.schedule), math.inf)

    fits_t = []
    grid = sorted({1.0, spec.t_ref} | {10 ** (e / 4) for e in range(-28, 1)})
    for t_ref in grid:
        rep = selector.validate_heuristic(scen, spec.machine, spec.topo, model, t_ref=t_ref, makespan_fn=makespan)
        regrets = [v.regret for v in rep.verdicts if v.regret is not None]
        fits_t.append({"t_ref": t_ref, "agree": sum(v.agree for v in rep.verdicts), "n": len(rep.verdicts),
                       "mean_regret": round(statistics.mean(regrets), 4) if regrets else None,
                       "mean_regret_on_mismatches": round(rep.mean_regret_on_mismatches, 4)})
    best = max(fits_t, key=lambda r: (r["agree"], -(r["mean_regret"] or 0), -abs(math.log10(r["t_ref"]))))
    default = next(r for r in fits_t if r["t_ref"] == 1.0)
    res = {"note": __doc__.split("\n\n")[0], "scenarios": table, "t_ref_grid": fits_t, "fitted": best,
           "reference_default": default, "machine_file_t_ref": spec.t_ref}
    print("fitted", best, "default", default, flush=True)
    with open(os.path.join(out_dir, "heuristic_sweep2.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

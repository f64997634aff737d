"""C5: the schedule heuristic vs the MEASURED exhaustive best over GEMM shapes (BASELINE.json configs[4]).

``selector.validate_heuristic`` (heuristic.py:74-115) with ``makespan_fn`` = measured makespans on
this B200 (``executor.MeasuredMakespan``: rank 0 of a virtual 8-rank job, L2 flushed, median of
10) instead of the simulator. Scenarios: the BASELINE configs that fit one GPU plus every corpus /
synthetic-grid scenario (data/scenarios_corpus.csv, cli_data.synthetic_grid) whose per-GPU GEMM
and buffers fit one B200 in seconds — skinny (M << N), square-ish, large-K and tall shapes.
The heuristic is scored twice on the same measurements: with the B200 machine file (fitted t_ref,
tools/calibrate.py) and with the reference's default t_ref = 1 s.
Writes <out>/heuristic_sweep.csv (export_report_csv, per t_ref) and <out>/heuristic_sweep.json.
usage: python tools/heuristic_sweep.py [out_dir]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_10236_b200 import machines, runtime, selector  # noqa: E402
from paper_2512_10236_b200.cli_data import synthetic_grid  # noqa: E402
from paper_2512_10236_b200.domain import parse_scenarios  # noqa: E402
from paper_2512_10236_b200.executor import MeasuredMakespan  # noqa: E402
from paper_2512_10236_b200.ops import _scenario  # noqa: E402
from importlib import resources  # noqa: E402

MAX_FLOPS = 1.2e14          # per-GPU GEMM work (~80 ms at B200 rates)
MAX_BYTES = 40e9            # gathered A (both parities) + output


def fits(sc) -> bool:
    g = sc.gemm
    return 2 * g.m * g.n * g.k <= MAX_FLOPS and 2 * (2 * g.m * g.k + g.m * g.n) <= MAX_BYTES


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    os.makedirs(out, exist_ok=True)
    runtime.load_library()
    spec = machines.b200_machine()
    model = machines.b200_calibration()
    scen = [_scenario("C2_llama3_8b_up", 8192, 3584, 4096, 8), _scenario("C1_bf16", 4096, 4096, 4096, 8),
            _scenario("C3p_llama3_70b_up", 16384, 7168, 8192, 8), _scenario("C4_cp_qk_T", 131072, 16384, 128, 8)]
    corpus = parse_scenarios(resources.files("paper_2512_10236_b200.data").joinpath("scenarios_corpus.csv")
                             .read_text())
    scen += [s for s in list(corpus) + list(synthetic_grid()) if fits(s)]
    mk = MeasuredMakespan(warmup=3, reps=10)

    def measured(plan):
        try:
            return mk(plan)
        except Exception as exc:  # e.g. uniform_fused_2d needs K/G to be a multiple of 64 here
            print(f"  {plan.scenario.name} {plan.schedule.value}: not executable ({exc})", flush=True)
            g = plan.scenario.gemm
            mk.cache[(g.m, g.n, g.k, plan.scenario.n_gpus, plan.schedule)] = math.inf
            return math.inf

    res = {"scenarios": [], "note": __doc__.split("\n\n")[0]}
    for label, t_ref in (("b200_fitted_t_ref", spec.t_ref), ("reference_default_t_ref_1s", 1.0)):
        rep = selector.validate_heuristic(scen, spec.machine, spec.topo, model, t_ref=t_ref, makespan_fn=measured)
        with open(os.path.join(out, f"heuristic_sweep_{label}.csv"), "w") as f:
            f.write(selector.export_report_csv(rep))
        res[label] = {"t_ref": t_ref, "agreement": sum(v.agree for v in rep.verdicts), "scenarios": len(rep.verdicts),
                      "accuracy": round(rep.accuracy, 4),
                      "mean_regret_on_mismatches": round(rep.mean_regret_on_mismatches, 4)}
        print(label, res[label], flush=True)
    for (m, n, k, g, kind), t in sorted(mk.cache.items(), key=lambda kv: (*kv[0][:4], kv[0][4].value)):
        res["scenarios"].append({"m": m, "n": n, "k": k, "kind": kind.value,
                                 "measured_us": None if math.isinf(t) else round(t * 1e6, 2)})
    with open(os.path.join(out, "heuristic_sweep.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

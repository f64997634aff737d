"""Generate golden fixtures by running the UNMODIFIED reference simulator.

The reference (/root/reference/pkg, ``overlap_sim`` 0.1.0) is pure Python,
so it is imported in place here (build container only; /root/reference does
not exist on the GPU box) and its outputs are frozen as JSON under
``tests/golden/``. Usage::

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Fixtures:
  plans_small.json    full task lists (every field) for small scenarios x all 7 kinds
  plans_digest.json   sha256 of the canonical task list for the large configs (C1-C4, g1, ...)
  selector.json       select_schedule over corpus + synthetic grid + configs + random shapes
  heuristic.json      validate_heuristic (speedups per kind, verdicts) on corpus + grid
  simulate.json       simulate() makespans, mesh/switch/example machines
  metrics.json        gemm_flops / gemm_mt / gemm_otb and lookup() KATs
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import random
import sys

from overlap_sim import core, heuristic, lossmodel, machines, planner
from overlap_sim.cli import synthetic_grid
from overlap_sim.engine import simulate

HERE = pathlib.Path(__file__).resolve().parent


def task_record(t) -> list:
    k = t.kind
    if isinstance(k, planner.TransferSpec):
        body = ["T", k.src, k.dst, k.bytes, int(k.fine), k.round_idx]
    elif isinstance(k, planner.GatherSpec):
        body = ["G", k.bytes]
    elif isinstance(k, planner.ScatterSpec):
        body = ["S", k.bytes]
    else:
        s = k.shape
        body = ["M", s.m, s.n, s.k, s.elt_bytes, int(k.additive),
                None if k.dil is None else [k.dil[0], repr(k.dil[1])],
                [list(f) for f in k.rows], None if k.col_block is None else list(k.col_block)]
    return [t.id, t.gpu, list(t.deps)] + body


def plan_record(plan) -> dict:
    return {"schedule": plan.schedule.value, "chunk_rows": plan.chunk_rows, "chunk_cols": plan.chunk_cols,
            "tasks": [task_record(t) for t in plan.tasks]}


def digest(rec: dict) -> str:
    return hashlib.sha256(json.dumps(rec, separators=(",", ":")).encode()).hexdigest()


def scen(name, m, n, k, g, elt=2):
    return core.Scenario(name=name, parallelism=core.Parallelism.SP_TP, model="golden",
                         gemm=core.GemmShape(m, n, k, elt), collective=core.Collective.ALL_GATHER, n_gpus=g)


# BASELINE.json configs as reference scenarios (SURVEY.md §8 notation line).
CONFIGS = [
    scen("C1", 4096, 4096, 4096, 4, 4),
    scen("C2", 8192, 3584, 4096, 8),
    scen("C2up", 8192, 1792, 4096, 8),
    scen("C3g2", 16384, 8192, 14336, 2),
    scen("C3g4", 16384, 8192, 7168, 4),
    scen("C3g8", 16384, 8192, 3584, 8),
    scen("C3p", 16384, 7168, 8192, 8),
    scen("C4", 131072, 16384, 128, 8),
]

SMALL = [
    scen("s_g2", 64, 48, 32, 2),
    scen("s_g4", 64, 40, 64, 4),
    scen("s_g4b", 512, 256, 384, 4),
    scen("s_g8", 512, 64, 128, 8),
    scen("s_g2k", 256, 64, 4, 2),
    scen("s_g2odd", 256, 64, 3, 2),
    scen("s_g4f32", 256, 128, 256, 4, 4),
    scen("gpu_g2", 1024, 512, 512, 2),
    scen("gpu_g4", 2048, 768, 1024, 4),
    scen("gpu_g8", 8192, 512, 1024, 8),
]


def all_plans(s) -> dict:
    out = {}
    for kind in planner.ALL_KINDS:
        try:
            out[kind.value] = plan_record(planner.build_plan(s, kind))
        except planner.PlanError as exc:
            out[kind.value] = {"error": str(exc)}
    return out


def main() -> int:
    corpus = core.parse_scenarios(
        (pathlib.Path(planner.__file__).parent / "data" / "scenarios_corpus.csv").read_text())
    grid = synthetic_grid()

    small = {s.name: {"scenario": [s.gemm.m, s.gemm.n, s.gemm.k, s.gemm.elt_bytes, s.n_gpus],
                      "plans": all_plans(s)} for s in SMALL}
    (HERE / "plans_small.json").write_text(json.dumps(small, separators=(",", ":")) + "\n")

    big = {}
    for s in CONFIGS + corpus[:2]:
        plans = all_plans(s)
        big[s.name] = {"scenario": [s.gemm.m, s.gemm.n, s.gemm.k, s.gemm.elt_bytes, s.n_gpus],
                       "digests": {k: (digest(v) if "tasks" in v else v) for k, v in plans.items()},
                       "n_tasks": {k: len(v.get("tasks", [])) for k, v in plans.items()}}
    (HERE / "plans_digest.json").write_text(json.dumps(big, indent=1) + "\n")

    rng = random.Random(2512_10236)
    rand = []
    while len(rand) < 300:
        g = rng.choice([2, 4, 8])
        m = g * g * rng.randint(1, 1 << 14)
        k = rng.choice([g * g * rng.randint(1, 1 << 14), rng.randint(1, 1 << 20)])
        n = rng.randint(1, 1 << 17)
        try:
            rand.append(scen(f"r{len(rand)}", m, n, k, g))
        except ValueError:
            continue
    machine_docs = {
        "mesh": machines.default_machine(),
        "example": machines.example_machine(),
        "b200": machines.machine_spec_from_dict({
            "topology": "switch", "n_gpus": 8, "link_bw": 110e9, "nic_bw": 770e9,
            "peak_flops": 1.6081e15, "mem_bw": 6.5329e12, "gemm_efficiency": 0.8284}),
    }
    sel = []
    for s in corpus + grid + CONFIGS + rand:
        for mname, spec in machine_docs.items():
            for t_ref in (1.0, 1e-3, 1e-4, 10.0):
                sel.append([s.gemm.m, s.gemm.n, s.gemm.k, s.gemm.elt_bytes, s.n_gpus, mname, t_ref,
                            heuristic.select_schedule(s, spec.machine, t_ref).value])
    (HERE / "selector.json").write_text(json.dumps({"cases": sel}, separators=(",", ":")) + "\n")

    model = lossmodel.default_calibration()
    heur = {}
    for label, scs, spec in (("corpus_mesh", corpus, machines.default_machine()),
                             ("grid_mesh", grid, machines.default_machine())):
        rep = heuristic.validate_heuristic(scs, spec.machine, spec.topo, model, spec.t_ref)
        heur[label] = {
            "accuracy": repr(rep.accuracy),
            "mean_regret": repr(rep.mean_regret_on_mismatches),
            "verdicts": [[v.scenario, v.chosen.value, v.best.value, int(v.agree),
                          None if v.regret is None else repr(v.regret),
                          {k.value: repr(x) for k, x in v.speedups.items()}] for v in rep.verdicts],
        }
    (HERE / "heuristic.json").write_text(json.dumps(heur, indent=1) + "\n")

    sims = []
    for mname in ("mesh", "example"):
        spec = machine_docs[mname]
        for s in SMALL[:4] + CONFIGS[:2] + corpus[:3]:
            if s.n_gpus != spec.topo.n_gpus:
                from overlap_sim.topology import Topology
                topo = Topology(kind=spec.topo.kind, n_gpus=s.n_gpus, link_bw=spec.topo.link_bw)
            else:
                topo = spec.topo
            for kind in planner.ALL_KINDS:
                try:
                    plan = planner.build_plan(s, kind)
                except planner.PlanError:
                    continue
                r = simulate(plan, spec.machine, topo, model)
                sims.append([s.name, mname, kind.value, repr(r.makespan), repr(r.max_work_rel_error),
                             {k: repr(v) for k, v in sorted(r.busy_time.items())}])
    # switch topology + noise variant
    sw = machines.machine_spec_from_dict({"topology": "switch", "n_gpus": 8, "link_bw": 64e9,
                                          "peak_flops": 1.3e15, "noise": 0.05})
    for kind in planner.ALL_KINDS:
        r = simulate(planner.build_plan(CONFIGS[1], kind), sw.machine, sw.topo, model, seed=3)
        sims.append(["C2", "switch_noise", kind.value, repr(r.makespan), repr(r.max_work_rel_error), {}])
    (HERE / "simulate.json").write_text(json.dumps({"cases": sims}, separators=(",", ":")) + "\n")

    met = {"shapes": [], "lookup": []}
    for s in corpus + CONFIGS:
        g = s.gemm
        met["shapes"].append([g.m, g.n, g.k, g.elt_bytes, core.gemm_flops(g), core.gemm_mt(g), repr(core.gemm_otb(g))])
    for key, tab in model.gemm_dil_tables.items():
        for x in (1.0, 300.0, 777.7, 1500.0, 3300.0, 7000.0, 1e6):
            met["lookup"].append(["gemm_dil." + key, x, repr(lossmodel.lookup(tab, x))])
    for x in (1e3, 1e6, 2e7, 1e8, 5e8, 1e10):
        met["lookup"].append(["comm_dil", x, repr(lossmodel.lookup(model.comm_dil_table, x))])
    (HERE / "metrics.json").write_text(json.dumps(met, indent=1) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())

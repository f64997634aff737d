"""Host-side mirror vs the reference simulator's frozen outputs (tests/golden/).

Pins: planner routing/task DAGs (planner.py:152-390), selector choices
(heuristic.py:25-43), exhaustive validation (heuristic.py:74-115), simulated
makespans (engine.py:117-297), static metrics (core.py:147-159) and loss-table
lookups (lossmodel.py:58-72).
"""
import pytest

import paper_2512_10236_b200 as ficco
from paper_2512_10236_b200 import machines, pricing, routing, selector, simulator
from paper_2512_10236_b200.cli_data import corpus, synthetic_grid

from _golden import digest, load, plan_record, scen

SMALL = load("plans_small.json")
DIGESTS = load("plans_digest.json")


@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_plans_field_for_field(name):
    m, n, k, elt, g = SMALL[name]["scenario"]
    s = scen(name, m, n, k, g, elt)
    for kind in routing.ALL_KINDS:
        want = SMALL[name]["plans"][kind.value]
        if "error" in want:
            with pytest.raises(routing.PlanError) as ei:
                routing.build_plan(s, kind)
            assert str(ei.value) == want["error"]
            continue
        got = plan_record(routing.build_plan(s, kind))
        assert got == want, (name, kind)


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_config_plans_digest(name):
    m, n, k, elt, g = DIGESTS[name]["scenario"]
    s = scen(name, m, n, k, g, elt)
    for kind in routing.ALL_KINDS:
        want = DIGESTS[name]["digests"][kind.value]
        if isinstance(want, dict):
            with pytest.raises(routing.PlanError):
                routing.build_plan(s, kind)
            continue
        plan = routing.build_plan(s, kind)
        assert len(plan.tasks) == DIGESTS[name]["n_tasks"][kind.value]
        assert digest(plan_record(plan)) == want, (name, kind)
        assert routing.validate_plan(plan) == []


def test_selector_matches_reference():
    mach = {"mesh": machines.default_machine(), "example": machines.example_machine(),
            "b200": machines.machine_spec_from_dict({
                "topology": "switch", "n_gpus": 8, "link_bw": 110e9, "nic_bw": 770e9,
                "peak_flops": 1.6081e15, "mem_bw": 6.5329e12, "gemm_efficiency": 0.8284})}
    cases = load("selector.json")["cases"]
    assert len(cases) > 1000
    for m, n, k, elt, g, mname, t_ref, want in cases:
        s = scen("x", m, n, k, g, elt)
        assert selector.select_schedule(s, mach[mname].machine, t_ref).value == want


@pytest.mark.parametrize("label", ["corpus_mesh", "grid_mesh"])
def test_validate_heuristic_matches_reference(label):
    gold = load("heuristic.json")[label]
    spec = machines.default_machine()
    scs = corpus() if label.startswith("corpus") else synthetic_grid()
    rep = selector.validate_heuristic(scs, spec.machine, spec.topo, pricing.default_calibration(), spec.t_ref)
    assert repr(rep.accuracy) == gold["accuracy"]
    assert repr(rep.mean_regret_on_mismatches) == gold["mean_regret"]
    for v, (name, chosen, best, agree, regret, gains) in zip(rep.verdicts, gold["verdicts"]):
        assert (v.scenario, v.chosen.value, v.best.value, int(v.agree)) == (name, chosen, best, agree)
        assert (None if v.regret is None else repr(v.regret)) == regret
        assert {k.value: repr(x) for k, x in v.speedups.items()} == gains


def test_simulate_makespans_bit_identical():
    from _golden import scen as mk
    small = load("plans_small.json")
    digs = load("plans_digest.json")
    shapes = {n: v["scenario"] for n, v in list(small.items()) + list(digs.items())}
    shapes.update({c.name: [c.gemm.m, c.gemm.n, c.gemm.k, c.gemm.elt_bytes, c.n_gpus] for c in corpus()})
    model = pricing.default_calibration()
    mach = {"mesh": machines.default_machine(), "example": machines.example_machine()}
    sw = machines.machine_spec_from_dict({"topology": "switch", "n_gpus": 8, "link_bw": 64e9,
                                          "peak_flops": 1.3e15, "noise": 0.05})
    for name, mname, kind, makespan, err, busy in load("simulate.json")["cases"]:
        m, n, k, elt, g = shapes[name]
        s = mk(name, m, n, k, g, elt)
        if mname == "switch_noise":
            r = simulator.simulate(routing.build_plan(s, routing.ScheduleKind(kind)), sw.machine, sw.topo, model, seed=3)
        else:
            spec = mach[mname]
            topo = spec.topo if g == spec.topo.n_gpus else pricing.Topology(spec.topo.kind, g, spec.topo.link_bw)
            r = simulator.simulate(routing.build_plan(s, routing.ScheduleKind(kind)), spec.machine, topo, model)
            assert {kk: repr(v) for kk, v in sorted(r.busy_time.items())} == busy
        assert repr(r.makespan) == makespan, (name, mname, kind)
        assert repr(r.max_work_rel_error) == err


def test_metrics_and_lookup():
    met = load("metrics.json")
    for m, n, k, elt, fl, mt, otb in met["shapes"]:
        g = ficco.GemmShape(m, n, k, elt)
        assert ficco.gemm_flops(g) == fl and ficco.gemm_mt(g) == mt and repr(ficco.gemm_otb(g)) == otb
    model = pricing.default_calibration()
    for key, x, want in met["lookup"]:
        tab = model.comm_dil_table if key == "comm_dil" else model.gemm_dil_tables[key.split(".")[1]]
        assert repr(pricing.lookup(tab, x)) == want


def test_reference_known_answers():
    # Values the reference's own tests pin (pkg/tests/test_core.py:31-48, test_cli.py:61,122-123).
    g1 = ficco.GemmShape(16384, 16384, 131072, 2)
    assert ficco.gemm_flops(g1) == 70_368_744_177_664
    assert ficco.gemm_mt(g1) == 9_126_805_504
    s = scen("g1", 16384, 16384, 131072, 8)
    spec = machines.example_machine()
    r = simulator.simulate(routing.build_plan(s, routing.ScheduleKind.SERIAL), spec.machine, spec.topo,
                           pricing.default_calibration())
    assert r.makespan == pytest.approx(78.757352e-3, rel=1e-6)
    for kind in routing.ALL_KINDS:
        plan = routing.build_plan(s, kind)
        assert routing.validate_plan(plan) == []
        ingress = sum(t.kind.bytes for t in plan.tasks
                      if isinstance(t.kind, routing.TransferSpec) and t.kind.dst == 0)
        assert ingress == 3_758_096_384


def test_error_types_match_reference():
    with pytest.raises(ValueError, match="elt_bytes"):
        ficco.GemmShape(1, 1, 1, 3)
    with pytest.raises(routing.PlanError, match="M=8"):
        routing.build_plan(scen("odd", 8, 16, 4096, 8), routing.ScheduleKind.UNIFORM_FUSED_1D)
    with pytest.raises(pricing.CalibrationError):
        pricing.load_calibration('{"bogus": 1}')
    with pytest.raises(ficco.ScenarioParseError, match="line 2"):
        ficco.parse_scenarios("name,parallelism,model,M,N,K,elt_bytes,collective,n_gpus\nx,SP+TP,m,1,2\n")
    with pytest.raises(ValueError, match="reduce_scatter|collective"):
        ficco.parse_scenarios("name,parallelism,model,M,N,K,elt_bytes,collective,n_gpus\n"
                              "x,SP+TP,m,64,64,64,2,reduce_scatter,2\n")

"""The measured executor (executor.execute, the real twin of the reference's engine.simulate,
/root/reference/pkg/src/overlap_sim/engine.py:117) for every op, and its trace in the reference's
export_trace_csv schema (engine.py:310-318), so measured and simulated timelines diff directly.

Per op and schedule: the output matches the oracle, every span lies inside the measured makespan,
the CSV parses with the reference header and the simulator's own trace of the same plan has the same
columns. AG / A2A / CP: one gemm span per GemmSpec task of this rank plus one span per arriving
transfer. RS: one span per piece of the schedule's adjoint routing (lowering.rs_pieces).
"""
import csv
import io
import math

import numpy as np
import pytest
import torch

from oracle import ficco_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1.6e-2, 1e-2
KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
         "uniform_fused_2d"]
HEADER = ["task_id", "gpu", "kind", "start_s", "end_s", "contended_fraction"]


def _t(x):
    return torch.from_numpy(x).to(torch.bfloat16).cuda()


def _np(t):
    return t.float().cpu().numpy()


@pytest.fixture(scope="module")
def mods():
    from paper_2512_10236_b200 import executor, machines, ops, routing, runtime, simulator
    runtime.load_library()
    return executor, machines, ops, routing, simulator


def _check_trace(res, plan, mods, n_spans):
    executor, machines, ops, routing, simulator = mods
    assert res.makespan > 0
    assert len(res.timeline) == n_spans
    for s in res.timeline:
        assert 0.0 <= s.start <= s.end <= res.makespan * 1.5, s  # trace clock vs event clock: loose bound
    rows = list(csv.reader(io.StringIO(simulator.export_trace_csv(res))))
    assert rows[0] == HEADER and len(rows) == n_spans + 1
    spec = machines.b200_machine()
    topo = type(spec.topo)(kind=spec.topo.kind, n_gpus=plan.scenario.n_gpus, link_bw=spec.topo.link_bw,
                           nic_bw=spec.topo.nic_bw, latency=spec.topo.latency)
    sim = simulator.simulate(plan, spec.machine, topo, machines.b200_calibration())
    assert list(csv.reader(io.StringIO(simulator.export_trace_csv(sim))))[0] == HEADER


def _ag_spans(plan, rank, routing):
    gemms = [t for t in plan.tasks if t.gpu == rank and isinstance(t.kind, routing.GemmSpec)
             and (t.kind.col_block is None or t.kind.col_block[0] == 0)]
    xfers = [t for t in plan.tasks if isinstance(t.kind, routing.TransferSpec) and t.kind.dst == rank]
    return len(gemms), len(xfers)


@pytest.mark.parametrize("kind", KINDS)
def test_execute_ag_trace(mods, kind):
    executor, machines, ops, routing, simulator = mods
    G, rank, R, K, N = 4, 1, 512, 1024, 512
    shards = [orc.seeded_inputs(21, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(21, 99, (N, K), "normal")
    _, outs = orc.execute_ag(kind, shards, w)
    plan = routing.build_plan(ops._scenario("ag", G * R, N, K, G), routing.ScheduleKind(kind))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, [_t(s) for s in shards])
        out, res = executor.execute(plan, _t(shards[rank]), _t(w), grp)
        np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
        n_gemm, n_xfer = _ag_spans(plan, rank, routing)
        gemm_spans = [s for s in res.timeline if s.kind == "gemm"]
        assert len(gemm_spans) == n_gemm
        # every arriving transfer gates some tile, except the 2D kind's later k-segments and the
        # serial kind (one gate for the whole gather): at least one landing per source
        assert 1 <= len(res.timeline) - n_gemm <= n_xfer
        _check_trace(res, plan, mods, len(res.timeline))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("agent", ["dma", "core"])
def test_execute_rs_trace(mods, kind, agent):
    executor, machines, ops, routing, simulator = mods
    from paper_2512_10236_b200.lowering import rs_pieces
    G, rank = 4, 2
    M, Kg, N = 128 * G * G, 256, 512
    a = [orc.seeded_inputs(22, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(22, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    sc = ops._scenario("rs", M, N, Kg, G)
    plan = routing.build_plan(sc, routing.ScheduleKind(kind))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent=agent)
        grp.load_peer_partials(low, [_t(x) for x in peers])
        out, res = executor.execute(plan, _t(a[rank]), _t(w[rank]), grp, op="rs", comm_agent=agent)
        np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
        order, _ = rs_pieces(sc, routing.ScheduleKind(kind), rank)
        assert [s.kind for s in res.timeline] == [f"gemm[->{pc.owner}]" if rem else "reduce" for rem, pc in order]
        _check_trace(res, plan, mods, len(order))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["serial", "shard_overlap_p2p", "hetero_unfused_1d"])
def test_execute_cp_and_a2a_trace(mods, kind):
    executor, machines, ops, routing, simulator = mods
    from paper_2512_10236_b200.domain import Collective
    G, rank, d, Tq, Tkv = 4, 3, 128, 256, 2048
    q = orc.seeded_inputs(23, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(23, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    plan = routing.build_plan(ops._scenario("cp", Tkv, Tq, d, G), routing.ScheduleKind(kind))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind)
        grp.load_peer_shards(low, [_t(x) for x in ks])
        out, res = executor.execute(plan, _t(q), _t(ks[rank]), grp, op="cp")
        np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
        n_gemm, _ = _ag_spans(plan, rank, routing)
        assert len([s for s in res.timeline if s.kind == "gemm"]) == n_gemm
        _check_trace(res, plan, mods, len(res.timeline))
    finally:
        grp.close()
    R, K, N = 256, 512, 256
    sends = [orc.seeded_inputs(24, p, (G * R, K)) for p in range(G)]
    wl = [orc.seeded_inputs(25, p, (N, K), "normal") for p in range(G)]
    _, outs = orc.execute_a2a(kind, sends, wl)
    sc = ops._scenario("a2a", G * R, N, K, G, Collective.ALL_TO_ALL)
    plan = routing.build_plan(sc, routing.ScheduleKind(kind))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_a2a(grp, R, K, N, kind)
        grp.load_peer_sends(low, [_t(sends[p][rank * R:(rank + 1) * R]) for p in range(G)])
        out, res = executor.execute(plan, _t(sends[rank]), _t(wl[rank]), grp, op="a2a")
        np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
        _check_trace(res, plan, mods, len(res.timeline))
    finally:
        grp.close()


def test_validate_heuristic_with_measured_makespans(mods):
    """The reference's validate_heuristic (heuristic.py:74-115) with makespan_fn = executor.MeasuredMakespan
    (real runs on this B200 instead of the simulator) on three small shapes: skinny, square-ish and M <= K."""
    executor, machines, ops, routing, simulator = mods
    from paper_2512_10236_b200 import selector
    scen = [ops._scenario("skinny", 4096, 1024, 512, 8), ops._scenario("square", 2048, 2048, 2048, 8),
            ops._scenario("m_le_k", 2048, 1024, 4096, 8)]
    spec = machines.b200_machine()
    mk = executor.MeasuredMakespan(warmup=2, reps=5)
    rep = selector.validate_heuristic(scen, spec.machine, spec.topo, machines.b200_calibration(), t_ref=spec.t_ref,
                                      makespan_fn=mk)
    assert len(rep.verdicts) == 3
    for sc, v in zip(scen, rep.verdicts):
        assert v.chosen is selector.select_schedule(sc, spec.machine, spec.t_ref)
        fine = {k: s for k, s in v.speedups.items() if k in routing.FINE_GRAIN_KINDS}
        assert fine and all(0 < s < 10 for s in fine.values()), v.speedups
        assert v.best is max(routing.FINE_GRAIN_KINDS, key=lambda k: v.speedups.get(k, float("-inf")))
        assert v.agree == (v.chosen is v.best) and (v.regret == 0.0 if v.agree else 0.0 < v.regret < 1.0)
    assert v.chosen is routing.ScheduleKind.UNIFORM_FUSED_2D  # M <= K
    assert {k for (*_, k) in mk.cache} >= set(routing.FINE_GRAIN_KINDS) | {routing.ScheduleKind.SERIAL}

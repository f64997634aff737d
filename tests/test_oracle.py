"""Pin the CPU oracle (oracle/ficco_oracle.py) to the reference's own outputs.

The oracle's routing restatement must reproduce, for every kind and every
golden scenario, the exact TransferSpec sequence and GemmSpec fragments the
reference planner emitted (tests/golden/plans_small.json); its selector must
reproduce every golden select_schedule case. Numerics (unpinned by the
reference) are checked for internal consistency: every schedule yields the
same gathered buffer (bit-exact) and the same product as one full matmul.
"""
import numpy as np
import pytest

from oracle import ficco_oracle as orc

from _golden import load

SMALL = load("plans_small.json")


@pytest.mark.parametrize("name", sorted(SMALL))
def test_oracle_routing_matches_reference(name):
    m, n, k, elt, g = SMALL[name]["scenario"]
    for kind in orc.KINDS:
        want = SMALL[name]["plans"][kind]
        if "error" in want:
            with pytest.raises(ValueError):
                orc.transfers(kind, m, k, g, elt)
            continue
        # task record: [id, gpu, deps, "T", src, dst, bytes, fine, round]
        ref_x = [(t[5], t[4], t[6], bool(t[7]), t[8]) for t in want["tasks"] if t[3] == "T"]
        assert orc.transfers(kind, m, k, g, elt) == ref_x, (name, kind)
        for gpu in range(g):
            # [id, gpu, deps, "M", m, n, k, elt, additive, dil, rows, col_block]
            ref_m = [(tuple(tuple(f) for f in t[10]), None if t[11] is None else tuple(t[11]))
                     for t in want["tasks"] if t[3] == "M" and t[1] == gpu]
            assert orc.gemm_fragments(kind, m, k, g, gpu) == ref_m, (name, kind, gpu)


def test_oracle_selector_matches_reference():
    peak = {"mesh": 1.3e15, "example": 1e15, "b200": 1.6081e15}
    for m, n, k, elt, g, mname, t_ref, want in load("selector.json")["cases"]:
        assert orc.select_schedule(m, n, k, peak[mname], t_ref) == want


def test_bf16_round_known_answers():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.140625, 1e-40, np.inf], dtype=np.float32)
    y = orc.bf16_round(x)
    # 1+2^-8 is a tie between 1 and 1+2^-7 -> even (1.0); 1.005859375 rounds up
    assert y[0] == 1.0 and y[1] == 1.0 and y[2] == np.float32(1.0078125)
    assert y[3] == -2.5 and y[4] == np.float32(3.140625) and y[6] == np.inf
    import torch
    r = np.random.default_rng(0).standard_normal(4096).astype(np.float32)
    ref = torch.from_numpy(r).to(torch.bfloat16).float().numpy()
    assert np.array_equal(orc.bf16_round(r), ref)


@pytest.mark.parametrize("g", [2, 4])
def test_oracle_schedules_agree(g):
    R, K, N = 32, 64, 48
    shards = [orc.seeded_inputs(0, p, (R, K)) for p in range(g)]
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    full = np.concatenate(shards)
    want = full @ w.T
    for kind in ("serial", "shard_overlap_p2p") + orc.FINE:
        gathered, outs = orc.execute_ag(kind, shards, w)
        for gpu in range(g):
            assert np.array_equal(gathered[gpu], full), (kind, gpu)
            np.testing.assert_allclose(outs[gpu], want, rtol=1e-5, atol=1e-5)


def test_oracle_rs_and_cp():
    g, M, Kg, N = 4, 64, 32, 40
    a = [orc.seeded_inputs(1, p, (M, Kg)) for p in range(g)]
    w = [orc.seeded_inputs(1, 100 + p, (N, Kg), "normal") for p in range(g)]
    outs = orc.execute_rs(a, w)
    full = sum(x @ y.T for x, y in zip(a, w))
    for q in range(g):
        np.testing.assert_allclose(outs[q], full[q * 16:(q + 1) * 16], rtol=2e-2, atol=2e-2)
    qm = orc.seeded_inputs(2, 0, (16, 32), "normal")
    ks = [orc.seeded_inputs(2, 1 + p, (8, 32), "normal") for p in range(g)]
    s, kall = orc.execute_cp_qk(qm, ks, 0.5)
    np.testing.assert_allclose(s, 0.5 * qm @ kall.T, rtol=1e-6)


@pytest.mark.parametrize("kind", orc.KINDS)
def test_a2a_dispatch_routes_each_block_to_its_rank(kind):
    """EP all-to-all (reference: planned like all-gather, collective inert): rank g's rows
    p*R.. hold peer p's block g, bit-exact, and C = dispatched @ W_g^T for every schedule."""
    G, R, K, N = 4, 64, 128, 32
    if kind == "ideal":
        pytest.skip("pricing bound, not an executable schedule")
    sends = [orc.seeded_inputs(3, p, (G * R, K)) for p in range(G)]
    ws = [orc.seeded_inputs(4, p, (N, K), "normal") for p in range(G)]
    try:
        disp, outs = orc.execute_a2a(kind, sends, ws)
    except ValueError:
        pytest.skip("kind not buildable at this shape")
    for g in range(G):
        want = np.concatenate([sends[p][g * R:(g + 1) * R] for p in range(G)])
        assert np.array_equal(disp[g], want)
        np.testing.assert_allclose(outs[g], want @ ws[g].T, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("kind", ["serial", "hetero_unfused_1d", "uniform_fused_2d"])
def test_a2a_rank_sample_computes_the_last_fragment(kind):
    """execute_a2a_rank (the EP CPU baseline) routes and computes every fragment into an R-row sink:
    after the call the sink holds the plan's last computed piece, equal to the same rows of execute_a2a."""
    G, R, K, N, g = 4, 64, 128, 32, 2
    sends = [orc.seeded_inputs(5, p, (G * R, K)) for p in range(G)]
    ws = [orc.seeded_inputs(6, p, (N, K), "normal") for p in range(G)]
    disp, _ = orc.execute_a2a(kind, sends, ws)
    blocks = [sends[p][g * R:(g + 1) * R] for p in range(G)]
    sink = orc.execute_a2a_rank(kind, blocks, ws[g], g)
    rows, col_block = orc.gemm_fragments(kind, G * R, K, G, g)[-1]
    if col_block is not None:  # the last K block's product for the last R rows
        k0, kb = col_block
        want = disp[g][-R:, k0:k0 + kb] @ ws[g][:, k0:k0 + kb].T
        np.testing.assert_allclose(sink, want, rtol=1e-5, atol=1e-4)
    else:
        start, count = rows[-1]
        last = list(range(start, start + count, R))[-1]
        n = min(R, start + count - last)
        np.testing.assert_allclose(sink[:n], disp[g][last:last + n] @ ws[g].T, rtol=1e-5, atol=1e-4)


def test_a2a_plans_equal_all_gather_plans():
    """The reference's planner never reads the collective: the product planner
    gives an EP all_to_all scenario the same task list as the all_gather scenario."""
    from paper_2512_10236_b200 import build_plan
    from paper_2512_10236_b200.domain import Collective
    from paper_2512_10236_b200.ops import _scenario
    from paper_2512_10236_b200.routing import supported_kinds
    ag = _scenario("x", 4096, 512, 1024, 8)
    ep = _scenario("x", 4096, 512, 1024, 8, Collective.ALL_TO_ALL)
    assert supported_kinds(ag) == supported_kinds(ep)
    for kind in supported_kinds(ag):
        a, e = build_plan(ag, kind), build_plan(ep, kind)
        assert [(t.gpu, t.deps, t.kind) for t in a.tasks] == [(t.gpu, t.deps, t.kind) for t in e.tasks], kind


C1_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
            "uniform_fused_2d"]


def test_c1_at_size_every_kind():
    """BASELINE.json configs[0] at its size: 4 simulated ranks, M = N = K = 4096, fp32, every executable
    schedule through the oracle (the reference's CPU sweep, /root/reference/pkg/tests/test_acceptance.py:87-118).

    Per rank and kind: the routed (gathered) operand is bit-exact, per-GPU ingress is (G-1)*R*K*e and the
    GEMM fragments cover 2MNK exactly (the reference's conservation criterion), and the result matches
    one full fp32 matmul (only the fragmenting / the 2D K-block summation order differs).
    """
    from paper_2512_10236_b200 import ops
    from paper_2512_10236_b200.routing import GemmSpec, ScheduleKind, TransferSpec, build_plan
    G, M, N, K, elt = 4, 4096, 4096, 4096, 4
    R = M // G
    shards = [orc.seeded_inputs(0, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    full = np.concatenate(shards)
    want = full @ w.T
    sc = ops._scenario("c1", M, N, K, G)
    sc = type(sc)(name=sc.name, parallelism=sc.parallelism, model=sc.model,
                  gemm=type(sc.gemm)(M, N, K, elt), collective=sc.collective, n_gpus=G)
    for kind in C1_KINDS:
        plan = build_plan(sc, ScheduleKind(kind))
        for gpu in range(G):
            ingress = sum(t.kind.bytes for t in plan.tasks if isinstance(t.kind, TransferSpec) and t.kind.dst == gpu)
            flops = sum(t.kind.flops for t in plan.tasks if t.gpu == gpu and isinstance(t.kind, GemmSpec))
            assert ingress == (G - 1) * R * K * elt and flops == 2 * M * N * K, (kind, gpu)
            assert sum(x[2] for x in orc.transfers(kind, M, K, G, elt) if x[0] == gpu) == ingress
        for gpu in (0, G - 1):
            buf, c = orc._route_and_gemm(kind, shards, w, gpu)
            assert np.array_equal(buf, full), kind
            np.testing.assert_allclose(c, want, rtol=1e-4, atol=1e-4, err_msg=kind)

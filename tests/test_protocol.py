"""Cross-rank protocol of the lowered programs, executed by the multi-rank interpreter (CPU).

Every executable schedule is lowered for every rank of a G-rank job and run
for several consecutive calls under randomised interleavings
(tests/protocol_sim.py). After each call each rank's outputs must match the
oracle: gathered buffers bit-exact, GEMM outputs within bf16 tolerance, RS
shards equal to the rank-ordered sum of partials. Stale or not-yet-written
bytes (a missing dependency, an early buffer reuse) show up as mismatches;
a missing signal shows up as a deadlock.
"""
import numpy as np
import pytest

from oracle import ficco_oracle as orc
from paper_2512_10236_b200.domain import Collective
from paper_2512_10236_b200.lowering import lower_ag, lower_rs
from paper_2512_10236_b200.ops import _scenario
from paper_2512_10236_b200.routing import ScheduleKind, build_plan

from paper_2512_10236_b200.runtime import OP_BARRIER
from protocol_sim import Deadlock, World, bf16_bits, bits_f32

AG_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
            "uniform_fused_2d"]
RUNS = 3


def _ag_world(kind, G, R, K, N, cta_group, seed):
    sc = _scenario("sim", R * G, N, K, G)
    lows = [lower_ag(build_plan(sc, ScheduleKind(kind)), g, "A", cta_group=cta_group) for g in range(G)]
    ws = max(low.ws_bytes for low in lows)
    for low in lows:
        low.ws_bytes = ws
    w = orc.seeded_inputs(seed, 999, (N, K), "normal")
    args, expect = [], []
    for run in range(RUNS):
        shards = [orc.seeded_inputs(seed * 10 + run, g, (R, K)) for g in range(G)]
        full = np.concatenate(shards)
        expect.append((full, full @ w.T))
        args.append([{"a": bf16_bits(shards[g]), "b": bf16_bits(w),
                      "c": np.zeros((R * G, N), dtype=np.uint16)} for g in range(G)])
    return lows, args, expect


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_ag_protocol(kind, G, cta_group):
    R, K, N = 64, 256, 64
    for seed in range(3):
        lows, args, expect = _ag_world(kind, G, R, K, N, cta_group, seed)
        world = World(lows, args, seed=seed)
        checked = []

        def on_done(rank, run, world=world):
            full, c_ref = expect[run]
            low = lows[rank]
            off = low.gather_off + (low.gather_par if run & 1 else 0)
            gat = world.ranks[rank].ws[off: off + full.size * 2].view(np.uint16).reshape(full.shape)
            assert np.array_equal(bits_f32(gat), full), (kind, rank, run, "gathered")
            c = bits_f32(args[run][rank]["c"])
            np.testing.assert_allclose(c, c_ref, rtol=2e-2, atol=2e-2, err_msg=f"{kind} rank {rank} run {run}")
            checked.append((rank, run))

        world.on_run_done = on_done
        world.run(RUNS)
        assert len(checked) == G * RUNS


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_a2a_protocol(kind, G, cta_group):
    """EP all-to-all -> expert GEMM: same plans as all-gather, per-destination payloads."""
    R, K, N = 64, 256, 64
    for seed in range(2):
        sc = _scenario("a2a", R * G, N, K, G, Collective.ALL_TO_ALL)
        lows = [lower_ag(build_plan(sc, ScheduleKind(kind)), g, "A", cta_group=cta_group) for g in range(G)]
        ws = max(low.ws_bytes for low in lows)
        for low in lows:
            low.ws_bytes = ws
        args, expect = [], []
        for run in range(RUNS):
            sends = [orc.seeded_inputs(seed * 10 + run, g, (R * G, K)) for g in range(G)]
            wl = [orc.seeded_inputs(seed * 10 + run, 50 + g, (N, K), "normal") for g in range(G)]
            expect.append(orc.execute_a2a(kind, sends, wl))
            args.append([{"a": bf16_bits(sends[g]), "b": bf16_bits(wl[g]),
                          "c": np.zeros((R * G, N), dtype=np.uint16)} for g in range(G)])
        world = World(lows, args, seed=seed)
        checked = []

        def on_done(rank, run, world=world):
            disp, outs = expect[run]
            low = lows[rank]
            off = low.gather_off + (low.gather_par if run & 1 else 0)
            full = disp[rank]
            gat = world.ranks[rank].ws[off: off + full.size * 2].view(np.uint16).reshape(full.shape)
            assert np.array_equal(bits_f32(gat), full), (kind, rank, run, "dispatched")
            np.testing.assert_allclose(bits_f32(args[run][rank]["c"]), outs[rank], rtol=2e-2, atol=2e-2,
                                       err_msg=f"{kind} rank {rank} run {run}")
            checked.append((rank, run))

        world.on_run_done = on_done
        world.run(RUNS)
        assert len(checked) == G * RUNS


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("agent", ["dma", "core", "nvls"])
def test_rs_protocol(kind, G, cta_group, agent):
    """comm_agent 'dma': copy-engine pushes of the partial pieces; 'core': the tile epilogues store
    the partials straight into the owners' receive slots and count tiles into their flag words.
    Every executable kind has an RS adjoint (lowering.rs_pieces), uniform_fused_2d as N blocks."""
    r, Kg = 16, 64
    N = 64 if kind != "uniform_fused_2d" else 32 * G
    M = r * G * G
    R = M // G
    for seed in range(3):
        sc = _scenario("rs", M, N, Kg, G)
        lows = [lower_rs(sc, ScheduleKind(kind), g, cta_group=cta_group, comm_agent=agent) for g in range(G)]
        ws = max(low.ws_bytes for low in lows)
        for low in lows:
            low.ws_bytes = ws
        args, expect = [], []
        for run in range(RUNS):
            a = [orc.seeded_inputs(seed * 10 + run, g, (M, Kg)) for g in range(G)]
            w = [orc.seeded_inputs(seed * 10 + run, 50 + g, (N, Kg), "normal") for g in range(G)]
            expect.append(orc.execute_rs(a, w, own_bf16=agent == "nvls"))
            args.append([{"a": bf16_bits(a[g]), "b": bf16_bits(w[g]), "c": np.zeros((R, N), dtype=np.uint16)}
                         for g in range(G)])
        world = World(lows, args, seed=seed)
        done = []

        def on_done(rank, run):
            np.testing.assert_allclose(bits_f32(args[run][rank]["c"]), expect[run][rank], rtol=2e-2, atol=3e-2,
                                       err_msg=f"{kind} rank {rank} run {run}")
            done.append(1)

        world.on_run_done = on_done
        world.run(RUNS)
        assert len(done) == G * RUNS


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "serial",
                                  "shard_overlap_p2p"])
@pytest.mark.parametrize("cta_group", [1, 2])
def test_cp_protocol(kind, cta_group):
    G, d, Tq, Tkv = 4, 64, 96, 512
    sc = _scenario("cp", Tkv, Tq, d, G)
    lows = [lower_ag(build_plan(sc, ScheduleKind(kind)), g, "B", alpha=0.125, other_rows=Tq, cta_group=cta_group)
            for g in range(G)]
    ws = max(low.ws_bytes for low in lows)
    for low in lows:
        low.ws_bytes = ws
    args, expect = [], []
    for run in range(RUNS):
        q = orc.seeded_inputs(run, 77, (Tq, d), "normal")
        ks = [orc.seeded_inputs(run, g, (Tkv // G, d), "normal") for g in range(G)]
        expect.append(orc.execute_cp_qk(q, ks, 0.125)[0])
        args.append([{"a": bf16_bits(q), "b": bf16_bits(ks[g]), "c": np.zeros((Tq, Tkv), dtype=np.uint16)}
                     for g in range(G)])
    world = World(lows, args, seed=7)

    def on_done(rank, run):
        np.testing.assert_allclose(bits_f32(args[run][rank]["c"]), expect[run], rtol=2e-2, atol=2e-2)

    world.on_run_done = on_done
    world.run(RUNS)


def test_missing_signal_deadlocks():
    """The interpreter really enforces gating: dropping a pull chain's signals must deadlock."""
    from paper_2512_10236_b200.runtime import OP_SIGNAL
    from protocol_sim import Deadlock
    lows, args, _ = _ag_world("hetero_unfused_1d", 2, 64, 256, 64, 1, 0)
    lows[1].ops = [op for op in lows[1].ops if op.op != OP_SIGNAL]
    with pytest.raises(Deadlock):
        World(lows, args).run(1)


@pytest.mark.parametrize("kind", AG_KINDS)
def test_ag_inplace_inputs(kind):
    """Zero-copy publish: each call's shard is written into the rank's own slot (parity of
    the call) by the caller just before the call; no local copy in the program."""
    G, R, K, N = 4, 64, 256, 64
    sc = _scenario("sim", R * G, N, K, G)
    for seed in range(2):
        lows = [lower_ag(build_plan(sc, ScheduleKind(kind)), g, "A", inplace=True) for g in range(G)]
        ws = max(low.ws_bytes for low in lows)
        for low in lows:
            low.ws_bytes = ws
        w = orc.seeded_inputs(seed, 999, (N, K), "normal")
        args, expect = [], []
        for run in range(RUNS):
            shards = [orc.seeded_inputs(seed * 10 + run, g, (R, K)) for g in range(G)]
            full = np.concatenate(shards)
            expect.append(full @ w.T)
            args.append([{"a": bf16_bits(shards[g]), "b": bf16_bits(w),
                          "c": np.zeros((R * G, N), dtype=np.uint16)} for g in range(G)])
        world = World(lows, args, seed=seed)

        def on_start(rank, run):
            low = lows[rank]
            off = low.gather_off + (low.gather_par if run & 1 else 0) + rank * R * K * 2
            world.ranks[rank].ws[off: off + R * K * 2] = args[run][rank]["a"].view(np.uint8).reshape(-1)

        def on_done(rank, run):
            np.testing.assert_allclose(bits_f32(args[run][rank]["c"]), expect[run], rtol=2e-2, atol=2e-2)

        world.on_run_start, world.on_run_done = on_start, on_done
        world.run(RUNS)


def test_rs_core_without_done_barrier_is_caught():
    """The direct-store RS relies on the DONE barrier before overwriting a peer's receive slot:
    dropping it (and the epilogue's go gate) lets a fast rank's next-run partials clobber a slow
    owner's slot before its reduction read it — the interpreter must see a wrong sum."""
    G, r, Kg, N = 3, 16, 64, 64
    M = r * G * G
    R = M // G
    bad = 0
    for seed in range(10):
        sc = _scenario("rs", M, N, Kg, G)
        lows = [lower_rs(sc, ScheduleKind.HETERO_FUSED_1D, g, cta_group=1, comm_agent="core") for g in range(G)]
        for low in lows:
            low.ops[:] = [op for op in low.ops if op.op != OP_BARRIER]
            low.desc.go_flag = 0
        ws = max(low.ws_bytes for low in lows)
        for low in lows:
            low.ws_bytes = ws
        args, expect = [], []
        for run in range(RUNS):
            a = [orc.seeded_inputs(seed * 10 + run, g, (M, Kg)) for g in range(G)]
            w = [orc.seeded_inputs(seed * 10 + run, 50 + g, (N, Kg), "normal") for g in range(G)]
            expect.append(orc.execute_rs(a, w))
            args.append([{"a": bf16_bits(a[g]), "b": bf16_bits(w[g]), "c": np.zeros((R, N), dtype=np.uint16)}
                         for g in range(G)])
        world = World(lows, args, seed=seed)
        wrong = []

        def on_done(rank, run):
            if not np.allclose(bits_f32(args[run][rank]["c"]), expect[run][rank], rtol=2e-2, atol=3e-2):
                wrong.append((rank, run))

        world.on_run_done = on_done
        try:
            world.run(RUNS)
        except (Deadlock, AssertionError):
            wrong.append("error")
        bad += bool(wrong)
    assert bad > 0


@pytest.mark.parametrize("split", [2, 3])
@pytest.mark.parametrize("G", [2, 4])
def test_ag_ring_split_protocol(split, G, monkeypatch):
    """The shard ring with each step's pull split over parallel copy streams (FICCO_RING_SPLIT):
    every part lands before RING[i] and before the right neighbour is notified."""
    monkeypatch.setenv("FICCO_RING_SPLIT", str(split))
    test_ag_protocol("shard_overlap_p2p", G, 2)


@pytest.mark.parametrize("split", [2, 3])
@pytest.mark.parametrize("G", [2, 4])
def test_ag_2d_slab_split_protocol(split, G, monkeypatch):
    """uniform_fused_2d with each R x b slab pulled as `split` row blocks on parallel copy streams
    (FICCO_2D_SPLIT): every part lands before the slab's XFER flag."""
    monkeypatch.setenv("FICCO_2D_SPLIT", str(split))
    test_ag_protocol("uniform_fused_2d", G, 2)


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "uniform_fused_2d"])
@pytest.mark.parametrize("G", [4, 8])
def test_ag_coalesced_rounds_protocol(kind, G, monkeypatch):
    """FICCO_COALESCE=1: consecutive rounds of one peer pulled by one copy ({0}, {1}, {2, 3}, {4..7}),
    every round's flag set right behind it; AG and all-to-all stay correct under random interleavings."""
    if kind == "uniform_fused_2d" and G == 8:
        pytest.skip("the interpreter's K = 256 gives K/G = 32, below the 64-column k-block")
    monkeypatch.setenv("FICCO_COALESCE", "1")
    test_ag_protocol(kind, G, 2)
    test_a2a_protocol(kind, G, 2)


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_unfused_1d"])
def test_cp_coalesced_rounds_protocol(kind, monkeypatch):
    monkeypatch.setenv("FICCO_COALESCE", "1")
    test_cp_protocol(kind, 2)

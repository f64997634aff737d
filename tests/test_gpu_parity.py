"""GPU parity: the CUDA path (C-ABI -> copy engines + tcgen05 tile kernel) vs the CPU oracle.

Bars: gathered buffers bit-exact; GEMM outputs (bf16 in, fp32
accumulate, bf16 out) within rtol=1.6e-2 / atol=1e-2 of the oracle's fp32
result (atol x sqrt(G) for RS).
"""
import math

import numpy as np
import pytest
import torch

from oracle import ficco_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1.6e-2, 1e-2


def _t(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(x).to(torch.bfloat16).cuda()


def _np(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


@pytest.fixture(scope="module")
def lib():
    from paper_2512_10236_b200 import runtime
    runtime.load_library()
    return runtime


@pytest.mark.parametrize("cfg", [(0, 1), (0, 2), (128, 1), (160, 2), (192, 2), (224, 2), (256, 2), (224, 1)])
@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (256, 512, 1024), (384, 544, 520), (1000, 96, 200),
                                   (2048, 3584, 4096)])
def test_tile_gemm_matches_fp32(lib, m, n, k, cfg):
    tile_n, cg = cfg
    a = orc.seeded_inputs(0, 0, (m, k))
    w = orc.seeded_inputs(0, 1, (n, k), "normal")
    out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    lib.gemm_bf16(_t(a), _t(w), out, tile_n=tile_n, cta_group=cg)
    torch.cuda.synchronize()
    np.testing.assert_allclose(_np(out), a @ w.T, rtol=RTOL, atol=ATOL)


def test_tile_gemm_alpha_and_grid(lib):
    a = orc.seeded_inputs(3, 0, (512, 256))
    w = orc.seeded_inputs(3, 1, (768, 256), "normal")
    out = torch.empty(512, 768, dtype=torch.bfloat16, device="cuda")
    lib.gemm_bf16(_t(a), _t(w), out, alpha=0.125, grid=7)
    torch.cuda.synchronize()
    np.testing.assert_allclose(_np(out), 0.125 * (a @ w.T), rtol=RTOL, atol=ATOL)


def test_cached_kernel_params_follow_alpha_and_knobs(lib, monkeypatch):
    """The library reuses a plan's kernel parameters while the call is unchanged: a new alpha on the same
    buffers, or a launch-time knob toggled between calls, must still take effect (bit-exact per setting)."""
    a = orc.seeded_inputs(4, 0, (512, 256))
    w = orc.seeded_inputs(4, 1, (512, 256), "normal")
    ta, tw = _t(a), _t(w)
    out = torch.empty(512, 512, dtype=torch.bfloat16, device="cuda")
    outs = {}
    for alpha in (1.0, 0.5, 1.0, 0.25):
        lib.gemm_bf16(ta, tw, out, alpha=alpha)
        torch.cuda.synchronize()
        np.testing.assert_allclose(_np(out), alpha * (a @ w.T), rtol=RTOL, atol=ATOL)
        if alpha in outs:
            assert torch.equal(outs[alpha], out)
        outs[alpha] = out.clone()
    for knob in ("0", "1", "0"):  # straight-line vs generic epilogue: same bits
        monkeypatch.setenv("FICCO_EPI_FAST", knob)
        lib.gemm_bf16(ta, tw, out)
        torch.cuda.synchronize()
        assert torch.equal(out, outs[1.0])


AG_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
            "uniform_fused_2d"]


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("G,rank,R,K,N", [(4, 0, 512, 1024, 768), (4, 3, 512, 1024, 768), (2, 1, 256, 512, 256),
                                          (8, 5, 128, 512, 512), (3, 2, 384, 768, 384), (6, 5, 384, 768, 256)])
def test_ag_virtual_matches_oracle(lib, kind, G, rank, R, K, N):
    from paper_2512_10236_b200 import ops
    shards = [orc.seeded_inputs(0, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag(kind, shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, [_t(s) for s in shards])
        a, wt = _t(shards[rank]), _t(w)
        for it in range(3):  # both workspace parities
            out, gathered = ops.all_gather_matmul(a, wt, kind=kind, group=grp, return_gathered=True)
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank]), (kind, it)
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d"])
def test_ag_ragged_chunks(lib, kind):
    """Chunks of 96 rows (tiles straddle nothing, partial 128-row boxes), N tail of 32, K tail of 8."""
    from paper_2512_10236_b200 import ops
    G, R, K, N = 4, 384, 520, 544
    shards = [orc.seeded_inputs(5, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(5, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag(kind, shards, w)
    grp = ops.FiccoGroup.virtual_group(G, 1)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, [_t(s) for s in shards])
        out, gathered = ops.all_gather_matmul(_t(shards[1]), _t(w), kind=kind, group=grp, return_gathered=True)
        grp.comm.check()
        assert np.array_equal(_np(gathered), gathered_ref[1])
        np.testing.assert_allclose(_np(out), outs[1], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


RS_KINDS = AG_KINDS  # every executable kind has an RS adjoint (lowering.rs_pieces); 2D = N blocks


@pytest.mark.parametrize("kind", RS_KINDS)
@pytest.mark.parametrize("G,rank", [(2, 0), (4, 2), (8, 7)])
def test_rs_virtual_matches_oracle(lib, kind, G, rank):
    from paper_2512_10236_b200 import ops
    M, Kg, N = 128 * G * G, 256, 512
    a = [orc.seeded_inputs(7, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(7, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind)
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind=kind, group=grp)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", RS_KINDS)
@pytest.mark.parametrize("agent", ["dma", "core"])
@pytest.mark.parametrize("G,rank", [(3, 1), (6, 4)])
def test_rs_odd_world_sizes_match_oracle(lib, kind, agent, G, rank):
    """GEMM -> RS with G = 3 and 6 ranks (flag blocks, receive slots and pair tiles at non-power-of-2 G)."""
    from paper_2512_10236_b200 import ops
    M, Kg, N = 128 * G * G, 256, 768
    a = [orc.seeded_inputs(25, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(25, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent=agent)
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind=kind, group=grp, comm_agent=agent)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "shard_overlap_p2p",
                                  "serial"])
def test_cp_qk_three_ranks_matches_oracle(lib, kind):
    """CP QK^T at G = 3 (kv chunks of 512 rows, non-power-of-2 world)."""
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 3, 2, 128, 384, 4608
    q = orc.seeded_inputs(27, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(27, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind)
        grp.load_peer_shards(low, [_t(x) for x in ks])
        for _ in range(2):
            out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind=kind, group=grp)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "serial"])
def test_cp_qk_virtual_matches_oracle(lib, kind):
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 1, 128, 384, 4096
    q = orc.seeded_inputs(9, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(9, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind)
        grp.load_peer_shards(low, [_t(x) for x in ks])
        for _ in range(2):
            out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind=kind, group=grp)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["shard_overlap_p2p", "hetero_unfused_1d", "uniform_fused_2d"])
def test_ag_input_slot_zero_copy(lib, kind):
    """Inputs produced directly in the group's symmetric slot skip the publish copy."""
    from paper_2512_10236_b200 import ops
    G, rank, R, K, N = 4, 2, 256, 512, 256
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        for call in range(3):
            shards = [orc.seeded_inputs(call, p, (R, K)) for p in range(G)]
            _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
            grp.load_peer_shards(low, [_t(s) for s in shards])
            slot = grp.input_slot(R, K, N, kind)
            slot.copy_(_t(shards[rank]))
            out, gathered = ops.all_gather_matmul(slot, _t(w), kind=kind, group=grp, return_gathered=True)
            grp.comm.check()
            assert ("ag", R * G, N, K, ops.ScheduleKind(kind), True, "dma") in grp._plans  # the in-place plan ran
            full = np.concatenate(shards)
            assert np.array_equal(_np(gathered), full)
            np.testing.assert_allclose(_np(out), full @ w.T, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["shard_overlap_p2p", "hetero_unfused_1d", "serial"])
def test_cp_kv_slot_zero_copy(lib, kind):
    """CP: a K shard produced in the group's symmetric slot (kv_slot) skips the publish copy; same scores."""
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 2, 128, 384, 4096
    q = orc.seeded_inputs(11, 50, (Tq, d), "normal")
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        for call in range(3):
            ks = [orc.seeded_inputs(20 + call, p, (Tkv // G, d), "normal") for p in range(G)]
            want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
            _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind)
            grp.load_peer_shards(low, [_t(x) for x in ks])
            slot = grp.kv_slot(Tq, d, Tkv, kind)
            slot.copy_(_t(ks[rank]))
            out = ops.cp_kv_all_gather_qk(_t(q), slot, kind=kind, group=grp)
            grp.comm.check()
            assert any(k[0] == "cp" and k[6] is True for k in grp._plans)  # the in-place plan ran
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
            ref = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind=kind, group=grp)  # copied-in path
            grp.comm.check()
            assert torch.equal(ref, out)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", AG_KINDS)
def test_ag_core_agent_matches_oracle(lib, kind):
    """comm_agent='core': the transfers run as SM copy kernels beside the tile kernel; same results."""
    from paper_2512_10236_b200 import ops
    G, rank, R, K, N = 4, 3, 512, 1024, 768
    shards = [orc.seeded_inputs(2, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(2, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag(kind, shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind, comm_agent="core")
        assert low.desc.hints & 2
        grp.load_peer_shards(low, [_t(s) for s in shards])
        for it in range(3):
            out, gathered = ops.all_gather_matmul(_t(shards[rank]), _t(w), kind=kind, group=grp,
                                                  return_gathered=True, comm_agent="core")
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank]), (kind, it)
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", RS_KINDS)
def test_rs_core_agent_matches_oracle(lib, kind):
    from paper_2512_10236_b200 import ops
    G, rank = 4, 2
    M, Kg, N = 128 * G * G, 256, 512
    a = [orc.seeded_inputs(8, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(8, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent="core")
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind=kind, group=grp, comm_agent="core")
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
        # the pushes really happened: every remote owner's receive slot holds our partial chunks
        # (GPU-rounded partials: within the GEMM tolerance of the fp32 product, not bit-equal)
        part = a[rank] @ w[rank].T
        for q in range(G):
            if q == rank:
                continue
            slot = rank if rank < q else rank - 1
            got = grp.ws_tensor(q, low.recv_off + slot * low.recv_slot, (R, N))
            np.testing.assert_allclose(_np(got), part[q * R:(q + 1) * R], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


def test_cp_core_agent_matches_oracle(lib):
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 1, 128, 384, 4096
    q = orc.seeded_inputs(9, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(9, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, "hetero_unfused_1d", comm_agent="core")
        grp.load_peer_shards(low, [_t(x) for x in ks])
        out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind="hetero_unfused_1d", group=grp, comm_agent="core")
        grp.comm.check()
        np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", AG_KINDS)
@pytest.mark.parametrize("G,rank,R,K,N", [(4, 2, 256, 512, 384), (8, 0, 128, 512, 256), (3, 1, 384, 768, 256)])
@pytest.mark.parametrize("agent", ["dma", "core"])
def test_a2a_virtual_matches_oracle(lib, kind, G, rank, R, K, N, agent):
    """EP all-to-all -> expert GEMM: dispatched tokens bit-exact, expert GEMM within tolerance."""
    from paper_2512_10236_b200 import ops
    sends = [orc.seeded_inputs(5, p, (G * R, K)) for p in range(G)]
    ws = [orc.seeded_inputs(6, p, (N, K), "normal") for p in range(G)]
    disp_ref, outs = orc.execute_a2a(kind, sends, ws)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_a2a(grp, R, K, N, kind, comm_agent=agent)
        grp.load_peer_sends(low, [_t(sends[p][rank * R:(rank + 1) * R]) for p in range(G)])
        a, wt = _t(sends[rank]), _t(ws[rank])
        for _ in range(3):  # both workspace parities
            out, disp = ops.all_to_all_matmul(a, wt, kind=kind, group=grp, return_gathered=True,
                                              comm_agent=agent)
            grp.comm.check()
            assert np.array_equal(_np(disp), disp_ref[rank]), kind
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


def test_typed_entry_points_check_the_plan_role(lib):
    """ficco_ag_gemm / _gemm_rs / _cp_qk / _a2a_gemm refuse a plan lowered for another op."""
    from paper_2512_10236_b200 import ops
    G, R, K, N = 4, 256, 256, 256
    grp = ops.FiccoGroup.virtual_group(G, 0)
    try:
        ag, _, _ = ops.prepare_ag(grp, R, K, N, "hetero_fused_1d")
        rs, _, _ = ops.prepare_rs(grp, G * R, K, N, "hetero_fused_1d")
        cp, _, _ = ops.prepare_cp(grp, R, 128, G * R, "uniform_fused_1d")
        a = torch.zeros(G * R, K, dtype=torch.bfloat16, device="cuda")
        w = torch.zeros(N, K, dtype=torch.bfloat16, device="cuda")
        c = torch.zeros(G * R, max(N, G * R), dtype=torch.bfloat16, device="cuda")
        for plan, wrong in ((ag, "gemm_rs"), (ag, "cp_qk"), (rs, "ag_gemm"), (rs, "a2a_gemm"), (cp, "ag_gemm"),
                            (cp, "gemm_rs")):
            with pytest.raises(ValueError, match="not lowered for this op"):  # FICCO_EINVAL
                plan.run_op(wrong, a, w, c)
        grp.comm.check()
    finally:
        grp.close()


def test_missing_transfer_times_out_as_deadlock_error(lib, monkeypatch):
    """A tile program whose readiness flags are never set (copy program dropped) aborts after
    FICCO_FLAG_TIMEOUT_S and surfaces as the reference's engine.DeadlockError."""
    import time
    from paper_2512_10236_b200 import ops
    from paper_2512_10236_b200.lowering import lower_ag
    from paper_2512_10236_b200.routing import ScheduleKind, build_plan
    from paper_2512_10236_b200.simulator import DeadlockError
    G, R, K, N = 4, 256, 256, 256
    grp = ops.FiccoGroup.virtual_group(G, 0)
    try:
        low = lower_ag(build_plan(ops._scenario("t", G * R, N, K, G), ScheduleKind.HETERO_UNFUSED_1D), 0, "A")
        grp.ensure_workspace(low.ws_bytes)
        plan = lib.Plan(grp.comm, low.desc, [], list(low.tiles))  # no copies: XFER flags never set
        a = torch.zeros(R, K, dtype=torch.bfloat16, device="cuda")
        w = torch.zeros(N, K, dtype=torch.bfloat16, device="cuda")
        c = torch.empty(G * R, N, dtype=torch.bfloat16, device="cuda")
        monkeypatch.setenv("FICCO_FLAG_TIMEOUT_S", "1")
        t0 = time.time()
        plan.run(a, w, c)
        with pytest.raises(DeadlockError, match=r"flag block \d, word 3\d\d"):  # names an XFER word (320..)
            grp.comm.check()
        assert time.time() - t0 < 30
        # the communicator is poisoned: later runs refuse up front instead of computing on stale chunks
        with pytest.raises(DeadlockError, match="poisoned"):
            plan.run(a, w, c)
        plan.close()
    finally:
        grp.close()


@pytest.mark.parametrize("agent", ["dma", "core"])
@pytest.mark.parametrize("kind", ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d"])
def test_rs_ragged_chunks(lib, kind, agent):
    """GEMM -> RS with 96-row fine chunks (REDUCE boxes straddle slots), a K tail of 8 and an N tail of 32."""
    from paper_2512_10236_b200 import ops
    G, rank = 4, 2
    M, Kg, N = 96 * G * G, 200, 544
    a = [orc.seeded_inputs(11, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(11, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent=agent)
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind=kind, group=grp, comm_agent=agent)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["hetero_unfused_1d", "uniform_fused_1d", "serial", "shard_overlap_p2p"])
@pytest.mark.parametrize("agent", ["dma", "core"])
def test_rs_ragged_large_w_row_groups(lib, kind, agent):
    """W of 33.7 MB (> 32 MiB: the RS tile program goes in row groups of 128-row blocks sweeping N) with
    96-row chunks, so groups and CTA pairs mix blocks of different pieces, and a K tail of 8."""
    from paper_2512_10236_b200 import ops
    from paper_2512_10236_b200.lowering import W_ROW_MAJOR_BYTES
    G, rank = 4, 1
    M, Kg, N = 96 * G * G, 2056, 8192
    assert N * Kg * 2 > W_ROW_MAJOR_BYTES
    a = [orc.seeded_inputs(21, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(21, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent=agent)
        assert low.desc.hints & 1  # FICCO_HINT_A_EVICT_LAST: the grouped raster pins A
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind=kind, group=grp, comm_agent=agent)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["hetero_unfused_1d", "hetero_fused_1d", "uniform_fused_1d", "shard_overlap_p2p"])
def test_ag_ragged_large_w_groups_span_gates(lib, kind):
    """AG->GEMM with W of 33.7 MB: row groups span fragments of different gates (96-row chunks, so CTA
    pairs and groups mix chunks of different peers); gathered bits and C vs the oracle."""
    from paper_2512_10236_b200 import ops
    G, rank, R, K, N = 4, 3, 96 * 4, 2056, 8192
    shards = [orc.seeded_inputs(23, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(23, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag(kind, shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, [_t(s) for s in shards])
        for _ in range(2):
            out, gathered = ops.all_gather_matmul(_t(shards[rank]), _t(w), kind=kind, group=grp,
                                                  return_gathered=True)
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank])
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind", ["shard_overlap_p2p", "hetero_unfused_1d"])
def test_cp_ragged(lib, kind):
    """CP QK^T with 96-row kv chunks and a query count that is not a multiple of the tile width."""
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 3, 128, 416, 96 * 16
    q = orc.seeded_inputs(12, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(12, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind)
        grp.load_peer_shards(low, [_t(x) for x in ks])
        out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind=kind, group=grp)
        grp.comm.check()
        np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("kind,G", [("hetero_unfused_1d", 8), ("uniform_fused_1d", 8), ("uniform_fused_2d", 4)])
def test_ag_coalesced_rounds_match_oracle(lib, kind, G, monkeypatch):
    """FICCO_COALESCE=1: consecutive rounds of a peer share one copy; gathered bits and C unchanged."""
    from paper_2512_10236_b200 import ops
    monkeypatch.setenv("FICCO_COALESCE", "1")
    rank, R, K, N = 1, 512, 512, 384
    shards = [orc.seeded_inputs(19, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(19, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag(kind, shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        n_groups = {8: 4, 4: 3}[G]
        assert sum(op.op == 0 for op in low.ops) == 1 + n_groups * (G - 1)  # publish + one copy per group
        grp.load_peer_shards(low, [_t(s) for s in shards])
        for _ in range(3):
            out, gathered = ops.all_gather_matmul(_t(shards[rank]), _t(w), kind=kind, group=grp,
                                                  return_gathered=True)
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank])
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("split", [2, 3])
def test_ag_2d_slab_split_matches_oracle(lib, split, monkeypatch):
    """uniform_fused_2d with each R x b slab pulled as `split` row blocks on parallel copy streams."""
    from paper_2512_10236_b200 import ops
    monkeypatch.setenv("FICCO_2D_SPLIT", str(split))
    G, rank, R, K, N = 4, 1, 384, 512, 512
    shards = [orc.seeded_inputs(17, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(17, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag("uniform_fused_2d", shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, "uniform_fused_2d")
        assert sum(op.op == 0 for op in low.ops) == 1 + split * G * (G - 1)  # publish + split parts per slab
        grp.load_peer_shards(low, [_t(s) for s in shards])
        for _ in range(3):
            out, gathered = ops.all_gather_matmul(_t(shards[rank]), _t(w), kind="uniform_fused_2d", group=grp,
                                                  return_gathered=True)
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank])
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("split", [2, 4])
def test_ag_ring_split_matches_oracle(lib, split, monkeypatch):
    """shard_overlap_p2p with each ring step pulled as `split` row blocks on parallel copy streams."""
    from paper_2512_10236_b200 import ops
    monkeypatch.setenv("FICCO_RING_SPLIT", str(split))
    G, rank, R, K, N = 8, 3, 384, 512, 512
    shards = [orc.seeded_inputs(13, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(13, 99, (N, K), "normal")
    gathered_ref, outs = orc.execute_ag("shard_overlap_p2p", shards, w)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, "shard_overlap_p2p")
        assert sum(op.op == 0 for op in low.ops) == 1 + split * (G - 1)  # publish + split pulls per step
        grp.load_peer_shards(low, [_t(s) for s in shards])
        for _ in range(3):
            out, gathered = ops.all_gather_matmul(_t(shards[rank]), _t(w), kind="shard_overlap_p2p", group=grp,
                                                  return_gathered=True)
            grp.comm.check()
            assert np.array_equal(_np(gathered), gathered_ref[rank])
            np.testing.assert_allclose(_np(out), outs[rank], rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


@pytest.mark.parametrize("agent", ["dma", "core"])
def test_rs_2d_ragged(lib, agent):
    """N-block (2D-adjoint) GEMM -> RS: 160-column blocks (tile-width tails inside each block), K tail of 8."""
    from paper_2512_10236_b200 import ops
    G, rank = 4, 1
    M, Kg, N = 128 * G, 200, 640
    a = [orc.seeded_inputs(14, p, (M, Kg)) for p in range(G)]
    w = [orc.seeded_inputs(14, 100 + p, (N, Kg), "normal") for p in range(G)]
    want = orc.execute_rs(a, w)[rank]
    R = M // G
    peers = [orc.bf16_round(a[p] @ w[p].T)[rank * R:(rank + 1) * R] for p in range(G) if p != rank]
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_rs(grp, M, Kg, N, "uniform_fused_2d", comm_agent=agent)
        grp.load_peer_partials(low, [_t(x) for x in peers])
        for _ in range(2):
            out = ops.matmul_reduce_scatter(_t(a[rank]), _t(w[rank]), kind="uniform_fused_2d", group=grp,
                                            comm_agent=agent)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL * math.sqrt(G))
    finally:
        grp.close()


def test_unsupported_kinds_raise_instead_of_substituting(lib):
    """No silent schedule rewrite: a kind the executor cannot run for this shape raises PlanError."""
    from paper_2512_10236_b200 import ops
    from paper_2512_10236_b200.routing import PlanError
    grp = ops.FiccoGroup.virtual_group(4, 0)
    try:
        with pytest.raises(PlanError, match="N/G"):  # 544 / 4 = 136 columns: not a multiple of 32
            ops.prepare_rs(grp, 128 * 4, 256, 544, "uniform_fused_2d")
        with pytest.raises(PlanError, match="multiple of 64"):  # d / G = 32: no whole k-block per round
            ops.prepare_cp(grp, 256, 128, 1024, "uniform_fused_2d")
        with pytest.raises(PlanError):
            ops.prepare_rs(grp, 128 * 4, 256, 512, "ideal")
    finally:
        grp.close()


def test_cp_2d_kblocks_matches_oracle(lib):
    """CP QK^T under uniform_fused_2d (d = 512, G = 4: one 128-column k-slab of every K shard per round)."""
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 2, 512, 256, 2048
    q = orc.seeded_inputs(15, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(15, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, "uniform_fused_2d")
        grp.load_peer_shards(low, [_t(x) for x in ks])
        for _ in range(2):
            out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind="uniform_fused_2d", group=grp)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


def test_op_boundary_validates_operands(lib):
    """Malformed call arguments raise ValueError before any pointer reaches the C-ABI."""
    from paper_2512_10236_b200 import ops
    G, R, K, N = 4, 256, 256, 256
    grp = ops.FiccoGroup.virtual_group(G, 0)
    bf = dict(dtype=torch.bfloat16, device="cuda")
    a, w = torch.zeros(R, K, **bf), torch.zeros(N, K, **bf)
    try:
        bad = [
            (lambda: ops.all_gather_matmul(a.float(), w, group=grp), "bfloat16"),
            (lambda: ops.all_gather_matmul(a, torch.zeros(N, K // 2, **bf), group=grp), "shape"),
            (lambda: ops.all_gather_matmul(a, w[:, :128], group=grp), "contiguous"),
            (lambda: ops.all_gather_matmul(torch.zeros(K, R, **bf).t(), w, group=grp), "contiguous"),
            (lambda: ops.all_gather_matmul(a, w, group=grp, out=torch.empty(R, N, **bf)), "shape"),
            (lambda: ops.all_gather_matmul(a, w, group=grp, out=torch.empty(G * R, N, device="cuda")), "bfloat16"),
            (lambda: ops.all_gather_matmul(a.cpu(), w, group=grp), "CUDA"),
            (lambda: ops.matmul_reduce_scatter(torch.zeros(G * R, K, **bf), torch.zeros(N, 64, **bf), group=grp),
             "shape"),
            (lambda: ops.matmul_reduce_scatter(torch.zeros(G * R, K, **bf), w, group=grp,
                                               out=torch.empty(G * R, N, **bf)), "shape"),
            (lambda: ops.cp_kv_all_gather_qk(torch.zeros(R, 128, **bf), torch.zeros(R, 64, **bf), group=grp),
             "shape"),
            (lambda: ops.all_to_all_matmul(torch.zeros(G * R, K, **bf), w.to(torch.float16), group=grp), "bfloat16"),
            (lambda: ops.all_gather_matmul(torch.zeros(R * K + 1, **bf)[1:].view(R, K), w, group=grp), "aligned"),
        ]
        for call, msg in bad:
            with pytest.raises(ValueError, match=msg):
                call()
        out = ops.all_gather_matmul(a, w, kind="hetero_fused_1d", group=grp)  # well-formed: runs
        grp.comm.check()
        assert out.shape == (G * R, N)
    finally:
        grp.close()


@pytest.mark.parametrize("m,n,k", [(512, 20480, 128), (384, 19200, 64), (256, 20480, 256), (640, 19968, 192)])
@pytest.mark.parametrize("b_resident", ["1", "0"])
def test_tile_gemm_short_k_b_stationary(lib, m, n, k, b_resident, monkeypatch):
    """Short K (store-bound): the plain GEMM rasters B-stationary waves (each CTA pair keeps one column
    block of B in smem for all of M, padded last wave) and the kernel reuses the resident B rows."""
    monkeypatch.setenv("FICCO_B_RESIDENT", b_resident)
    a = orc.seeded_inputs(16, 0, (m, k))
    w = orc.seeded_inputs(16, 1, (n, k), "normal")
    out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    lib.gemm_bf16(_t(a), _t(w), out, alpha=0.5)
    torch.cuda.synchronize()
    np.testing.assert_allclose(_np(out), 0.5 * (a @ w.T), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("kind", ["shard_overlap_p2p", "uniform_fused_1d", "hetero_unfused_1d", "serial"])
@pytest.mark.parametrize("agent", ["dma", "core"])
def test_cp_b_stationary_waves(lib, kind, agent):
    """CP QK^T with more kv blocks than CTA pairs (80 units: one full wave of 74 + a padded partial wave):
    the B-stationary tile order with resident K rows, gated per fragment, matches the oracle."""
    from paper_2512_10236_b200 import ops
    G, rank, d, Tq, Tkv = 4, 1, 128, 512, 20480
    q = orc.seeded_inputs(17, 50, (Tq, d), "normal")
    ks = [orc.seeded_inputs(17, p, (Tkv // G, d), "normal") for p in range(G)]
    want, _ = orc.execute_cp_qk(q, ks, 1.0 / math.sqrt(d))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind, comm_agent=agent)
        assert sum(t.rows == 0 for t in low.tiles) > 0  # the padded wave is there
        grp.load_peer_shards(low, [_t(x) for x in ks])
        for _ in range(2):
            out = ops.cp_kv_all_gather_qk(_t(q), _t(ks[rank]), kind=kind, group=grp, comm_agent=agent)
            grp.comm.check()
            np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL)
    finally:
        grp.close()


def test_nvls_fails_cleanly_or_reduces_in_the_switch(lib):
    """comm_agent='nvls' (in-switch reduction). Virtual peers share one device, so the
    op raises PlanError there. The multicast primitives either report the fabric's refusal as
    FICCO_ENODEV (NotImplementedError) or, where a one-device multicast object can be created, the
    multimem.ld_reduce kernel returns exactly the bound memory (the sum over one device)."""
    from paper_2512_10236_b200 import ops
    from paper_2512_10236_b200.routing import PlanError
    import ctypes as C
    grp = ops.FiccoGroup.virtual_group(4, 0)
    try:
        with pytest.raises(PlanError, match="real ranks"):
            ops.prepare_rs(grp, 128 * 16, 256, 512, "hetero_fused_1d", comm_agent="nvls")
    finally:
        grp.close()
    L = lib.load_library()
    if not lib.multicast_supported(0):
        h, mapped = C.c_void_p(), C.c_size_t()
        with pytest.raises(NotImplementedError, match="NVLS multicast unavailable"):
            lib.check(L.ficco_mc_create(64 << 20, 1, C.byref(h), C.byref(mapped)))
        return
    h, mapped = C.c_void_p(), C.c_size_t()
    lib.check(L.ficco_mc_create(8 << 20, 1, C.byref(h), C.byref(mapped)))
    try:
        lib.check(L.ficco_mc_add_device(h))
        uc, va = C.c_void_p(), C.c_void_p()
        lib.check(L.ficco_mc_bind(h, C.byref(uc), C.byref(va)))
        rows, cols = 512, 1024
        src = ops._wrap_device_ptr(uc.value, (rows, cols), torch.bfloat16)
        src.copy_(_t(orc.seeded_inputs(18, 0, (rows, cols))))
        out = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")
        lib.check(L.ficco_mc_reduce_bf16(va, C.c_void_p(out.data_ptr()), rows, cols, cols, cols,
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        assert torch.equal(out, src)
    finally:
        lib.check(L.ficco_mc_release(h))


@pytest.mark.parametrize("cta_group", [1, 2])
def test_mixed_tile_widths_in_one_program(lib, cta_group):
    """Per-tile UMMA widths: every tile of a lowered AG plan re-split into narrower tiles of mixed widths
    (32 / 64 / 96 / 128 inside a TN = 256 kernel) still matches the oracle (CTA-pair B split at
    cols/2, per-tile instruction descriptor)."""
    from paper_2512_10236_b200 import lowering, ops
    from paper_2512_10236_b200.runtime import Plan
    G, R, K, N = 4, 256, 512, 768
    shards = [orc.seeded_inputs(9, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(9, 99, (N, K), "normal")
    _, outs = orc.execute_ag("hetero_unfused_1d", shards, w)
    grp = ops.FiccoGroup.virtual_group(G, 2)
    try:
        _, low, _ = ops.prepare_ag(grp, R, K, N, "hetero_unfused_1d")
        grp.load_peer_shards(low, [_t(s) for s in shards])
        low = lowering.lower_ag(ops.build_plan(ops._scenario("ag", G * R, N, K, G),
                                               ops.ScheduleKind("hetero_unfused_1d")), 2, "A",
                                cta_group=cta_group)
        low.desc.tile_n = 256  # the widest kernel; every tile below is narrower
        widths = [64, 96, 128]
        tiles = []
        for i in range(0, len(low.tiles), cta_group):
            grp_t = low.tiles[i:i + cta_group]
            w0 = grp_t[0].cols
            cut = widths[(i // cta_group) % 3] if w0 > widths[(i // cta_group) % 3] else w0
            for off, cw in ((0, cut), (cut, w0 - cut)):
                if cw <= 0:
                    continue
                for t in grp_t:
                    tiles.append(lowering._tile(t.a_row, t.b_row + off, t.c_row, t.c_col + off, t.rows, cw, t.flag,
                                                t.fmask, t.kseg, t.kstride, t.mode, t.chunk, t.recv_row, t.a_src,
                                                t.b_src))
        assert len({t.cols for t in tiles}) >= 3
        plan = Plan(grp.comm, low.desc, low.ops, tiles)
        try:
            out = torch.empty(G * R, N, dtype=torch.bfloat16, device="cuda")
            for _ in range(2):
                plan.run(_t(shards[2]), _t(w), out)
                grp.comm.check()
                np.testing.assert_allclose(_np(out), outs[2], rtol=RTOL, atol=ATOL)
        finally:
            plan.close()
    finally:
        grp.close()

"""GPU parity at BASELINE.json's full sizes (C2, C4 and the EP corpus case at G = 8, C3 at G = 2, 4, 8; virtual peers
on one B200).

The CPU oracle cannot run these shapes in seconds, so the checks are the size-independent
properties of the path:

* routing: the gathered operand is bit-exact against the concatenation of the shards;
* schedule independence: every schedule kind and both comm agents give BIT-IDENTICAL
  outputs. Each output element is accumulated over K in the same k-block order by the same
  tcgen05 instruction shape, and RS sums the partials in the same rank order, so any
  routing or gating error shows up as a mismatch;
* identity with the flag-free tile GEMM of the gathered operand (AG / CP);
* idempotence: consecutive calls (alternating workspace parities) give identical results;
* numerics: the WHOLE output against a plain PyTorch fp32 reference of the same op (cuBLAS
  fp32 GEMM, TF32 off, computed in row blocks), and sampled rows from every shard against the
  oracle's fp32 arithmetic on the same bf16 inputs (numpy), both within the stated tolerance
  rtol 1.6e-2 / atol 1e-2 (x sqrt(G) for RS).
"""
import math

import numpy as np
import pytest
import torch

from oracle import ficco_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1.6e-2, 1e-2
G = 8
AG_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
            "uniform_fused_2d"]
RS_KINDS = AG_KINDS  # every executable kind has an RS adjoint (2D: N blocks)
CP_KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d"]


@pytest.fixture(scope="module")
def ops():
    from paper_2512_10236_b200 import ops as _ops
    from paper_2512_10236_b200 import runtime
    runtime.load_library()
    return _ops


def _rand(shape, seed, kind="uniform"):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if kind == "uniform":
        x = torch.rand(shape, generator=g, device="cuda") * 2 - 1
    else:
        x = torch.randn(shape, generator=g, device="cuda") / math.sqrt(shape[-1])
    return x.to(torch.bfloat16)


def _np(t):
    return t.float().cpu().numpy()


def _assert_close_fp32(out, a, w, alpha=1.0, addends=(), atol=ATOL, block=8192):
    """Every element of out [M, N] against alpha * a @ w^T (+ sum of addends) computed in fp32 by cuBLAS
    with TF32 off, in row blocks (C4's fp32 reference alone would be 8.6 GB)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        wf = w.float()
        for r0 in range(0, out.shape[0], block):
            ref = torch.matmul(a[r0:r0 + block].float(), wf.t())
            if alpha != 1.0:
                ref.mul_(alpha)
            for x in addends:
                ref += x[r0:r0 + block].float()
            got = out[r0:r0 + block].float()
            if not torch.allclose(got, ref, rtol=RTOL, atol=atol):
                err = ((got - ref).abs() - RTOL * ref.abs()).max().item()
                raise AssertionError(f"rows {r0}..: exceeds rtol {RTOL} / atol {atol} by {err}")
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _sample_rows(total, per_block, blocks, seed=0):
    """Rows spread over every shard: first, last and random rows of each of `blocks` blocks."""
    rng = np.random.default_rng(seed)
    size = total // blocks
    rows = []
    for b in range(blocks):
        rows += [b * size, b * size + size - 1] + list(b * size + rng.integers(1, size - 1, per_block - 2))
    return np.array(sorted(set(rows)))


@pytest.mark.parametrize("rank", [0, 5])
def test_c2_full_size_all_kinds_bit_identical(ops, rank):
    """C2: Llama-3-8B MLP up-proj AG->GEMM, (M, N, K) = (8192, 3584, 4096), G = 8."""
    from paper_2512_10236_b200 import runtime
    R, K, N = 1024, 4096, 3584
    shards = [_rand((R, K), 100 + p) for p in range(G)]
    w = _rand((N, K), 99, "normal")
    a_all = torch.cat(shards)
    plain = torch.empty(G * R, N, dtype=torch.bfloat16, device="cuda")
    runtime.gemm_bf16(a_all, w, plain)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        for agent in ("dma", "core"):
            for kind in AG_KINDS:
                _, low, _ = ops.prepare_ag(grp, R, K, N, kind, comm_agent=agent)
                grp.load_peer_shards(low, shards)
                for it in range(2):  # both workspace parities
                    out, gathered = ops.all_gather_matmul(shards[rank], w, kind=kind, group=grp,
                                                          return_gathered=True, comm_agent=agent)
                    grp.comm.check()
                    assert torch.equal(gathered, a_all), (agent, kind, it, "gathered operand")
                    assert torch.equal(out, plain), (agent, kind, it, "output differs from the plain GEMM")
    finally:
        grp.close()
    _assert_close_fp32(plain, a_all, w)
    rows = _sample_rows(G * R, 4, G)
    want = _np(a_all[rows]) @ _np(w).T
    np.testing.assert_allclose(_np(plain[rows]), want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("world", [8, 4, 2])
def test_c3_full_size_all_kinds_bit_identical(ops, world):
    """C3: Llama-3-70B down-proj GEMM->RS, (M, N, K/G) = (16384, 8192, 28672 / G) at G = 2, 4, 8, rank 0."""
    G = world
    rank, M, Kg, N = 0, 16384, 28672 // G, 8192
    R = M // G
    a = _rand((M, Kg), 200)
    w = _rand((N, Kg), 201, "normal")
    # the virtual peers' bf16 partials of this rank's rows (their A_g[rows q] @ W_g^T)
    peers = []
    for p in range(G):
        if p != rank:
            ap, wp = _rand((R, Kg), 300 + p), _rand((N, Kg), 400 + p, "normal")
            peers.append(torch.matmul(ap.float(), wp.float().t()).to(torch.bfloat16))
    grp = ops.FiccoGroup.virtual_group(G, rank)
    first = None
    try:
        for agent in ("dma", "core"):
            for kind in RS_KINDS:
                _, low, _ = ops.prepare_rs(grp, M, Kg, N, kind, comm_agent=agent)
                grp.load_peer_partials(low, peers)
                for it in range(2):
                    out = ops.matmul_reduce_scatter(a, w, kind=kind, group=grp, comm_agent=agent)
                    grp.comm.check()
                    if first is None:
                        first = out.clone()
                    else:
                        assert torch.equal(out, first), (agent, kind, it, "RS output differs between schedules")
    finally:
        grp.close()
    _assert_close_fp32(first, a[rank * R:(rank + 1) * R], w, addends=peers, atol=ATOL * math.sqrt(G))
    # oracle arithmetic on sampled rows: own fp32 partial + peers' bf16 partials in rank order
    rows = _sample_rows(R, 6, 4)
    acc = _np(a[rank * R + rows]) @ _np(w).T
    for part in peers:
        acc = acc + _np(part[rows])
    np.testing.assert_allclose(_np(first[rows]), acc, rtol=RTOL, atol=ATOL * math.sqrt(G))


def test_c4_full_size_all_kinds_bit_identical(ops):
    """C4: CP KV all-gather -> QK^T, 128K context, d = 128, 16384 local queries, G = 8 (4 GiB scores)."""
    from paper_2512_10236_b200 import runtime
    rank, Tq, d, Tkv = 2, 16384, 128, 131072
    q = _rand((Tq, d), 500, "normal")
    ks = [_rand((Tkv // G, d), 600 + p, "normal") for p in range(G)]
    k_all = torch.cat(ks)
    scale = 1.0 / math.sqrt(d)
    plain = torch.empty(Tq, Tkv, dtype=torch.bfloat16, device="cuda")
    runtime.gemm_bf16(q, k_all, plain, alpha=scale)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    out = torch.empty_like(plain)
    try:
        for agent in ("dma", "core"):
            for kind in CP_KINDS:
                _, low, _ = ops.prepare_cp(grp, Tq, d, Tkv, kind, comm_agent=agent)
                grp.load_peer_shards(low, ks)
                for it in range(2):
                    out.fill_(0)
                    ops.cp_kv_all_gather_qk(q, ks[rank], kind=kind, group=grp, out=out, comm_agent=agent)
                    grp.comm.check()
                    assert torch.equal(out, plain), (agent, kind, it, "scores differ from the plain GEMM")
    finally:
        grp.close()
    _assert_close_fp32(plain, q, k_all, alpha=scale, block=4096)
    rows = _sample_rows(Tq, 4, 8)
    want, _ = orc.execute_cp_qk(_np(q[rows]), [_np(k) for k in ks], scale)
    np.testing.assert_allclose(_np(plain[rows]), want, rtol=RTOL, atol=ATOL)


def test_ep_full_size_all_kinds_bit_identical(ops):
    """EP (corpus g14, Mixtral): all-to-all dispatch -> expert GEMM, (M, N, K) = (147456, 28672, 4096), G = 8."""
    from paper_2512_10236_b200 import runtime
    rank, M, N, K = 3, 147456, 28672, 4096
    R = M // G
    send = _rand((M, K), 700)
    blocks = [send[rank * R:(rank + 1) * R] if p == rank else _rand((R, K), 800 + p) for p in range(G)]
    w = _rand((N, K), 701, "normal")
    disp_ref = torch.cat(blocks)
    plain = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    runtime.gemm_bf16(disp_ref, w, plain)
    out = torch.empty_like(plain)
    grp = ops.FiccoGroup.virtual_group(G, rank)
    try:
        for agent in ("dma", "core"):
            for kind in AG_KINDS:
                _, low, _ = ops.prepare_a2a(grp, R, K, N, kind, comm_agent=agent)
                grp.load_peer_sends(low, blocks)
                for it in range(2):
                    out.fill_(0)
                    _, disp = ops.all_to_all_matmul(send, w, kind=kind, group=grp, out=out, return_gathered=True,
                                                    comm_agent=agent)
                    grp.comm.check()
                    assert torch.equal(disp, disp_ref), (agent, kind, it, "dispatched tokens")
                    assert torch.equal(out, plain), (agent, kind, it, "expert GEMM differs from the plain GEMM")
    finally:
        grp.close()
    _assert_close_fp32(plain, disp_ref, w)
    rows = _sample_rows(M, 3, G)
    np.testing.assert_allclose(_np(plain[rows]), _np(disp_ref[rows]) @ _np(w).T, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("agent", ["dma", "core"])
def test_c1_all_kinds_vs_oracle(ops, agent):
    """BASELINE.json configs[0] on the GPU: 4 ranks, M = N = K = 4096 (bf16 here; the CPU oracle runs it in
    fp32, tests/test_oracle.py::test_c1_at_size_every_kind), every executable schedule, every rank, against
    the oracle's execute_ag of the same bf16-valued inputs: gathered operand bit-exact, the whole product
    within rtol 1.6e-2 / atol 1e-2."""
    Gc, R, K, N = 4, 1024, 4096, 4096
    shards = [orc.seeded_inputs(0, p, (R, K)) for p in range(Gc)]
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    full = np.concatenate(shards)
    want = full @ w.T  # every kind's oracle output equals the full product up to fp32 summation order
    ts = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in shards]
    wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    for rank in range(Gc):
        grp = ops.FiccoGroup.virtual_group(Gc, rank)
        try:
            for kind in AG_KINDS:
                gathered_ref, outs = orc.execute_ag(kind, shards, w) if rank == 0 else (None, None)
                if rank == 0:  # the oracle's own per-kind result (fragment order, 2D K blocks) is the product
                    np.testing.assert_allclose(outs[0], want, rtol=1e-4, atol=1e-4)
                _, low, _ = ops.prepare_ag(grp, R, K, N, kind, comm_agent=agent)
                grp.load_peer_shards(low, ts)
                out, gathered = ops.all_gather_matmul(ts[rank], wt, kind=kind, group=grp, return_gathered=True,
                                                      comm_agent=agent)
                grp.comm.check()
                assert np.array_equal(_np(gathered), full), (kind, rank)
                np.testing.assert_allclose(_np(out), want, rtol=RTOL, atol=ATOL, err_msg=f"{kind} rank {rank}")
        finally:
            grp.close()

"""Full-size multi-rank parity on one B200: real processes, real arrival-gated reduction.

The virtual mode (one process) pre-lands every peer's partial before the run, so the
owner's REDUCE tiles never wait. Here G processes share cuda:0 and each is one rank of
a G-rank job at BASELINE.json's full sizes:

* C3 (Llama-3-70B down-proj GEMM -> reduce-scatter, seq 16384): (M, N, K) = (16384, 8192,
  28672/G) at G = 2 and 4, every executable RS schedule x {dma pushes, core epilogue stores}.
  The owner's tiles really wait for the peers' copy-engine pushes / remote TMA stores.
* C2-shaped AG at G = 2 (Llama-3-8B up-proj, seq 8192: N = 2 * 14336 / 2, K = 4096).

Checks, per rank and call:
* the WHOLE output against a plain PyTorch fp32 reference of the same op (cuBLAS fp32,
  TF32 off): the owner's fp32 partial plus the peers' bf16-rounded partials, rank order
  (the oracle's reduction order, oracle/ficco_oracle.py:execute_rs). Each peer's partial is
  rounded to bf16 on its own GPU after ITS fp32 accumulation, so a reference that rounds a
  differently-ordered fp32 sum may land one bf16 ulp of |P_g| away: the RS bound is therefore
  elementwise atol*sqrt(G) + rtol * sum_g |P_g| (the magnitude of the terms, not of their sum);
* sampled rows x columns against the numpy oracle's reduction (oracle.bf16_round, execute_rs's order);
* AG: the gathered buffer bit-exact (torch.equal) against the concatenated shards.

Inputs come from per-rank torch generators on the GPU, so every process can regenerate
any peer's operands. Tolerances: rtol 1.6e-2, atol 1e-2 * sqrt(G) (RS), 1e-2 (AG).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
         "uniform_fused_2d"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rs_operands(torch, g, M, K, N, call):
    ga = torch.Generator(device="cuda").manual_seed(7000 + 10 * g + call)
    gw = torch.Generator(device="cuda").manual_seed(8000 + 10 * g + call)
    a = (torch.rand(M, K, generator=ga, device="cuda") * 2 - 1).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=gw, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    return a, w


def _worker(rank, world, port, q, what):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from oracle import ficco_oracle as orc
    from paper_2512_10236_b200 import ops
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    errors = []
    try:
        grp = ops.FiccoGroup.distributed()
        if what == "rs":
            M, N, K = 16384, 8192, 28672 // world
            R = M // world
            own = slice(rank * R, (rank + 1) * R)
            sample = np.r_[0:4, R // 2:R // 2 + 4, R - 4:R]  # first / middle / last rows of the shard
            for call in range(2):
                ops_g = [_rs_operands(torch, g, M, K, N, call) for g in range(world)]
                # fp32 torch reference of this rank's shard (owner fp32 + peers' bf16 partials, rank order)
                ref = ops_g[rank][0][own].float() @ ops_g[rank][1].float().T
                mag = ref.abs()
                for g in range(world):
                    if g != rank:
                        p_g = (ops_g[g][0][own].float() @ ops_g[g][1].float().T).to(torch.bfloat16).float()
                        ref += p_g
                        mag += p_g.abs()
                # numpy oracle on sampled rows: execute_rs's formula on the owner's rows
                cols = np.r_[0:32, N // 2:N // 2 + 16, N - 16:N]
                a_s = [ops_g[g][0][own][sample].float().cpu().numpy() for g in range(world)]
                w_s = [ops_g[g][1][cols].float().cpu().numpy() for g in range(world)]
                want = a_s[rank] @ w_s[rank].T
                mag_s = np.abs(want)
                for g in range(world):
                    if g != rank:
                        p_g = orc.bf16_round(a_s[g] @ w_s[g].T)
                        want = want + p_g
                        mag_s = mag_s + np.abs(p_g)
                a, w = ops_g[rank]
                del ops_g
                for agent in ("dma", "core"):
                    for kind in KINDS:
                        print(f"rank {rank}: RS {kind} {agent} call {call}", flush=True)
                        out = ops.matmul_reduce_scatter(a, w, kind=kind, group=grp, comm_agent=agent)
                        grp.comm.check()
                        atol = 1e-2 * math.sqrt(world)
                        excess = ((out.float() - ref).abs() - (atol + 1.6e-2 * mag)).max().item()
                        if excess > 0:
                            errors.append(f"RS {kind} {agent} call {call}: output vs fp32 reference exceeds the "
                                          f"bound by {excess}")
                        got = out[sample][:, cols].float().cpu().numpy()
                        if (np.abs(got - want) > atol + 1.6e-2 * mag_s).any():
                            errors.append(f"RS {kind} {agent} call {call}: sampled rows vs the oracle")
                del a, w, ref, mag
                torch.cuda.empty_cache()
        else:  # C2-shaped AG at G = world
            M, N, K = 8192, 2 * 14336 // world, 4096
            R = M // world
            gw = torch.Generator(device="cuda").manual_seed(99)
            w = (torch.randn(N, K, generator=gw, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
            for call in range(2):
                shards = []
                for g in range(world):
                    gen = torch.Generator(device="cuda").manual_seed(1000 + 10 * g + call)
                    shards.append((torch.rand(R, K, generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16))
                full = torch.cat(shards)
                ref = full.float() @ w.float().T
                sample = np.r_[0:4, R - 4:R + 4, M - 4:M]
                want = full[sample].float().cpu().numpy() @ w.float().cpu().numpy().T
                for agent in ("dma", "core"):
                    for kind in KINDS:
                        print(f"rank {rank}: AG {kind} {agent} call {call}", flush=True)
                        out, gathered = ops.all_gather_matmul(shards[rank], w, kind=kind, group=grp,
                                                              return_gathered=True, comm_agent=agent)
                        grp.comm.check()
                        if not torch.equal(gathered, full):
                            errors.append(f"AG {kind} {agent} call {call}: gathered buffer differs")
                        if not torch.allclose(out.float(), ref, rtol=1.6e-2, atol=1e-2):
                            errors.append(f"AG {kind} {agent} call {call}: output vs fp32 reference")
                        if not np.allclose(out[sample].float().cpu().numpy(), want, rtol=1.6e-2, atol=1e-2):
                            errors.append(f"AG {kind} {agent} call {call}: sampled rows vs the oracle")
        grp.close()
    except Exception:
        errors.append(traceback.format_exc())
    q.put((rank, errors))
    dist.destroy_process_group()


def _run(world, what):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, what)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, errs = q.get(timeout=900)
            results[r] = errs
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert results.get(r) == [], f"rank {r}: {results.get(r, 'no result (hung or crashed)')}"


@pytest.mark.parametrize("world", [2, 4])
def test_c3_fullsize_reduce_scatter_real_ranks(world):
    _run(world, "rs")


def test_c2_fullsize_all_gather_real_ranks():
    _run(2, "ag")

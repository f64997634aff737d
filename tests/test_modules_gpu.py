"""The torch modules over the FiCCO ops (paper_2512_10236_b200/modules.py), forward AND backward, with real
ranks: G processes share cuda:0 (gloo for the handle exchange, CUDA-IPC workspaces), each one rank of a
tensor/sequence-parallel MLP block

    H = SequenceParallelColumnLinear(X_shard)   AG -> GEMM     (backward: GEMM -> RS)
    Y_shard = SequenceParallelRowLinear(H)      GEMM -> RS     (backward: AG -> GEMM)

checked against the same block computed unsharded in fp32 by plain PyTorch on every rank: the output
shard, dX_shard and both weight gradients, by relative Frobenius error (bf16 activations in between:
tolerance 3e-2). Schedules: the selector's default and explicit ones for both directions.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, kinds):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2512_10236_b200 import modules, ops
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    errors = []
    try:
        grp = ops.FiccoGroup.distributed()
        M, D, F = 128 * world * world, 256, 256 * world  # tokens, model dim, MLP hidden (F/G per rank)
        R, Fl = M // world, F // world
        g = torch.Generator(device="cuda").manual_seed(5)
        x = (torch.rand(M, D, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        w_up = (torch.randn(F, D, generator=g, device="cuda") / D ** 0.5).to(torch.bfloat16)
        w_down = (torch.randn(D, F, generator=g, device="cuda") / F ** 0.5).to(torch.bfloat16)
        gy = torch.randn(M, D, generator=g, device="cuda").to(torch.bfloat16)  # upstream gradient
        # the unsharded block in fp32 (every rank can rebuild it: same seeds)
        xr = x.float().requires_grad_(True)
        wur, wdr = w_up.float().requires_grad_(True), w_down.float().requires_grad_(True)
        yr = (xr @ wur.t()) @ wdr.t()
        (yr * gy.float()).sum().backward()

        def rel(a, b):
            return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-6))

        for fwd_kind, bwd_kind in kinds:
            col = modules.SequenceParallelColumnLinear(D, Fl, grp, kind=fwd_kind, backward_kind=bwd_kind,
                                                       device="cuda")
            row = modules.SequenceParallelRowLinear(Fl, D, grp, kind=fwd_kind, backward_kind=bwd_kind,
                                                    device="cuda")
            with torch.no_grad():
                col.weight.copy_(w_up[rank * Fl:(rank + 1) * Fl])
                row.weight.copy_(w_down[:, rank * Fl:(rank + 1) * Fl].contiguous())
            xs = x[rank * R:(rank + 1) * R].clone().requires_grad_(True)
            for it in range(2):  # consecutive calls: both workspace parities
                for p in (col.weight, row.weight, xs):
                    p.grad = None
                y = row(col(xs))
                (y * gy[rank * R:(rank + 1) * R]).sum().backward()
                grp.comm.check()
                tag = f"fwd {fwd_kind} bwd {bwd_kind} call {it}"
                checks = {
                    "Y_shard": (y, yr[rank * R:(rank + 1) * R]),
                    "dX_shard": (xs.grad, xr.grad[rank * R:(rank + 1) * R]),
                    "dW_up": (col.weight.grad, wur.grad[rank * Fl:(rank + 1) * Fl]),
                    "dW_down": (row.weight.grad, wdr.grad[:, rank * Fl:(rank + 1) * Fl]),
                }
                for name, (got, want) in checks.items():
                    e = rel(got, want)
                    if not e < 3e-2:
                        errors.append(f"{tag}: {name} relative error {e:.3e}")
        dist.barrier()
        grp.close()
    except Exception:
        errors.append(traceback.format_exc())
    q.put((rank, errors))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kinds", [
    (2, [(None, None), ("hetero_unfused_1d", "shard_overlap_p2p"), ("uniform_fused_2d", "serial")]),
    (4, [(None, None), ("shard_overlap_p2p", "hetero_fused_1d")]),
])
def test_tp_sp_mlp_block_forward_backward(world, kinds):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kinds)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, errs = q.get(timeout=600)
            results[r] = errs
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert results.get(r) == [], f"rank {r}: {results.get(r, 'no result (hung or crashed)')}"

"""Debug the multi-process (ranks sharing one GPU) protocol: phase timestamps per rank."""
import os
import socket
import sys
import time

import torch.multiprocessing as mp


def worker(rank, world, port, mode):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if mode == "serialize":
        os.environ["FICCO_SERIALIZE"] = "1"
    import torch
    import torch.distributed as dist
    from paper_2512_10236_b200 import ops
    t0 = time.time()
    log = lambda m: print(f"[r{rank} {time.time()-t0:6.2f}s] {m}", flush=True)  # noqa: E731
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grp = ops.FiccoGroup.distributed()
    R, K, N = 256, 512, 256
    a = torch.randn(R, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(R * world, N, dtype=torch.bfloat16, device="cuda")
    M, Kg = 64 * world * world, 256
    a2 = torch.randn(M, Kg, device="cuda").to(torch.bfloat16)
    w2 = torch.randn(N, Kg, device="cuda").to(torch.bfloat16)
    for opname, kind in [("ag", k) for k in ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d",
                                              "hetero_unfused_1d", "uniform_fused_2d"]] + \
                        [("rs", k) for k in ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d"]]:
        for call in range(2):
            if opname == "ag":
                ops.all_gather_matmul(a, w, kind=kind, group=grp, out=out)
            else:
                ops.matmul_reduce_scatter(a2, w2, kind=kind, group=grp)
            torch.cuda.synchronize()
            log(f"{opname} {kind} call {call} done")
    grp.comm.check()
    log("checked")
    dist.barrier()
    grp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ps = [ctx.Process(target=worker, args=(r, world, port, mode)) for r in range(world)]
    for p in ps:
        p.start()
    deadline = time.time() + 60
    for p in ps:
        p.join(timeout=max(1, deadline - time.time()))
    for p in ps:
        if p.is_alive():
            print("killing", p.pid, flush=True)
            p.kill()
    print("exitcodes", [p.exitcode for p in ps])

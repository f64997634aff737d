"""A/B of the shard ring's per-step pull split over parallel copy streams (FICCO_RING_SPLIT).

C2 (virtual 8 ranks, rank 0, zero-copy publish like the bench): shard_overlap_p2p plans lowered
with split = 1, 2, 4 timed interleaved step by step (bench.time_interleaved, L2 flushed before
every call), plus each plan's copy program alone (empty tile list, graph replay).
usage: python tools/ring_split_ab.py [steps]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import lowering, ops, runtime  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind, build_plan  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    runtime.load_library()
    G, M, N, K = 8, 8192, 3584, 4096
    R = M // G
    gen = torch.Generator(device="cuda").manual_seed(0)
    shards = [(torch.rand(R, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(G)]
    w = (torch.randn(N, K, generator=gen, device="cuda") / 64).to(torch.bfloat16)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    grp = ops.FiccoGroup.virtual_group(G, 0)
    sc = ops._scenario("c2", M, N, K, G)
    plans, copy_plans = {}, {}
    for split in (1, 2, 4):
        os.environ["FICCO_RING_SPLIT"] = str(split)
        low = lowering.lower_ag(build_plan(sc, ScheduleKind.SHARD_OVERLAP_P2P), 0, "A", inplace=True)
        grp.ensure_workspace(low.ws_bytes)
        grp.load_peer_shards(low, shards)
        for par in (0, 1):
            grp.ws_tensor(0, low.gather_off + par * low.gather_par, (R, K)).copy_(shards[0])
        plans[split] = runtime.Plan(grp.comm, low.desc, low.ops, low.tiles)
        copy_plans[split] = runtime.Plan(grp.comm, low.desc, low.ops, [])
    os.environ.pop("FICCO_RING_SPLIT")
    fns = [lambda p=p: p.run(shards[0], w, out) for p in plans.values()]
    fns += [lambda p=p: p.run(shards[0], w, out) for p in copy_plans.values()]
    times = bench.time_interleaved(fns, steps, 5, lambda: flush.fill_(1), torch.cuda.current_stream())
    grp.comm.check()
    names = [f"op split={s}" for s in plans] + [f"copy program alone split={s}" for s in copy_plans]
    for n, t in zip(names, times):
        print(f"{n:32s} median {statistics.median(t) * 1e3:7.1f} us", flush=True)
    for p in list(plans.values()) + list(copy_plans.values()):
        p.close()
    grp.close()


if __name__ == "__main__":
    main()

"""Back-to-back runs of one schedule with L2 flushes in between; check every `every` runs."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

runtime.load_library()
kind = sys.argv[1] if len(sys.argv) > 1 else "hetero_unfused_1d"
M, N, K = (int(x) for x in (sys.argv[2:5] if len(sys.argv) >= 5 else (8192, 3584, 4096)))
G = 8
R = M // G
shards = [(torch.rand(R, K, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(G)]
w = (torch.randn(N, K, device="cuda") / 64).to(torch.bfloat16)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grp = ops.FiccoGroup.virtual_group(G, 0)
_, low, _ = ops.prepare_ag(grp, R, K, N, kind)
grp.load_peer_shards(low, shards)
t0 = time.time()
for i in range(60):
    flush.fill_(1)
    ops.all_gather_matmul(shards[0], w, kind=kind, group=grp, out=out)
    if i % 5 == 4:
        try:
            grp.comm.check()
            print(f"run {i} ok {time.time()-t0:.2f}s", flush=True)
        except Exception as exc:
            print(f"run {i} FAILED: {exc}", flush=True)
            break

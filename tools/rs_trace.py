"""Measured timeline of the C3 GEMM->RS op (virtual 8 ranks): op latency vs tile-kernel span.

For each schedule: event-timed op latency (graph path), the tile kernel's span
(%globaltimer: first CTA start -> last tile stored), and, per epilogue mode
(STORE_SIGNAL = remote partial chunks, REDUCE = own chunk + peers' partials),
the mean tile duration (loads may start -> accumulator stored) and the time
the last such tile finished.
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import ops, runtime  # noqa: E402
from paper_2512_10236_b200.runtime import EPI_REDUCE, EPI_STORE_REMOTE, EPI_STORE_SIGNAL  # noqa: E402


def main():
    runtime.load_library()
    G, M, N, K = 8, 16384, 8192, 3584
    R = M // G
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = (torch.rand(M, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=gen, device="cuda") / 60).to(torch.bfloat16)
    out = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    grp = ops.FiccoGroup.virtual_group(G, 0)
    res = {}
    for kind in sys.argv[1:] or ["hetero_fused_1d", "uniform_fused_1d"]:
        agent = os.environ.get("RS_AGENT", "dma")
        plan, low, _ = ops.prepare_rs(grp, M, K, N, kind, comm_agent=agent)
        info = plan.info()
        trace = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device="cuda")
        plan.set_trace(trace)
        for _ in range(3):
            ops.matmul_reduce_scatter(a, w, kind=kind, group=grp, out=out, comm_agent=agent)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.fill_(1)
            x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x.record()
            ops.matmul_reduce_scatter(a, w, kind=kind, group=grp, out=out, comm_agent=agent)
            y.record()
            y.synchronize()
            ts.append(x.elapsed_time(y) * 1e3)
        grp.comm.check()
        tr = trace.cpu().tolist()
        g = info["grid"]
        t0 = min(tr[:g])
        ready = [(tr[g + 2 * i] - t0) / 1e3 for i in range(info["tiles"])]
        done = [(tr[g + 2 * i + 1] - t0) / 1e3 for i in range(info["tiles"])]
        modes = {}
        # CTA-pair tile lists interleave the two halves; group by the epilogue mode
        tiles = low.tiles
        for name, mode in (("store_signal", EPI_STORE_SIGNAL), ("store_remote", EPI_STORE_REMOTE),
                           ("reduce", EPI_REDUCE)):
            idx = [i for i, t in enumerate(tiles) if t.mode == mode]
            if not idx:
                continue
            dur = [done[i] - ready[i] for i in idx]
            modes[name] = {"n": len(idx), "mean_tile_us": round(statistics.mean(dur), 2),
                           "first_ready": round(min(ready[i] for i in idx), 1),
                           "last_done": round(max(done[i] for i in idx), 1)}
        res[kind] = {"op_us": round(statistics.median(ts), 1), "kernel_span_us": round(max(done), 1),
                     "cta_start_spread_us": round((max(tr[:g]) - t0) / 1e3, 1), "modes": modes}
        plan.set_trace(None)
    print(json.dumps(res, indent=1))
    grp.close()


if __name__ == "__main__":
    main()

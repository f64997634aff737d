"""A/B of the output-store L2 policy (FICCO_B_RESIDENT=1|0) on the plain tile GEMM and the C4 op,
interleaved call by call (same clocks), L2 flushed between calls. usage: python tools/out_hint_ab.py"""
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def rnd(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, generator=g, device="cuda") / math.sqrt(shape[-1])).to(torch.bfloat16)


def main():
    runtime.load_library()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cases = {}
    q, k = rnd((16384, 128), 1), rnd((131072, 128), 2)
    s = torch.empty(16384, 131072, dtype=torch.bfloat16, device="cuda")
    cases["c4_plain"] = lambda: runtime.gemm_bf16(q, k, s, alpha=0.088)
    cases["c4_cublas"] = lambda: torch.addmm(s, q, k.T, beta=0, alpha=0.088, out=s)
    G = 8
    grp = ops.FiccoGroup.virtual_group(G, 0)
    shards = [k[i * 16384:(i + 1) * 16384] for i in range(G)]
    for kind in ("shard_overlap_p2p", "hetero_unfused_1d"):
        _, low, _ = ops.prepare_cp(grp, 16384, 128, 131072, kind)
        grp.load_peer_shards(low, shards)
        cases[f"c4_op_{kind}"] = (lambda kd: lambda: ops.cp_kv_all_gather_qk(q, shards[0], kind=kd, group=grp,
                                                                            out=s))(kind)
    a2, w2 = rnd((8192, 4096), 3), rnd((3584, 4096), 4)
    c2 = torch.empty(8192, 3584, dtype=torch.bfloat16, device="cuda")
    cases["c2_plain"] = lambda: runtime.gemm_bf16(a2, w2, c2)
    a3, w3 = rnd((16384, 3584), 5), rnd((8192, 3584), 6)
    c3 = torch.empty(16384, 8192, dtype=torch.bfloat16, device="cuda")
    cases["c3_plain"] = lambda: runtime.gemm_bf16(a3, w3, c3)
    res = {}
    for name, fn in cases.items():
        times = {"1": [], "0": []}
        for rep in range(18):
            for mode in ("1", "0"):
                os.environ["FICCO_B_RESIDENT"] = mode
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if rep >= 3:
                    times[mode].append(e0.elapsed_time(e1) * 1e3)
        res[name] = {m: round(statistics.median(v), 1) for m, v in times.items()}
        print(name, res[name], flush=True)
    grp.close()
    with open(os.path.join(ROOT, "gpurun_out", "bres_ab.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

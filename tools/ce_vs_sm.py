"""Which agent executes a same-device copy: a copy engine, or an SM copy kernel?

Every SM is occupied for T ms (ficco_occupy_sms: 1 CTA x 1024 threads with the
full shared memory per SM, so no other CTA can be resident); a copy is issued
on another stream right after. If the copy's end event lands before T, a copy
engine ran it; if it lands after T, it waited for SMs. Variants: cudaMemcpyAsync
(1D), cudaMemcpy2DAsync, a ficco_copy_batch list, and the AG copy program of a virtual-peer FiCCO plan.
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

MiB = 1 << 20


def cudart():
    import glob
    import nvidia.cuda_runtime as m  # torch's bundled runtime
    libs = glob.glob(os.path.join(list(m.__path__)[0], "lib", "libcudart.so.*"))
    return C.CDLL(libs[0])


def probe(issue, occupy_ms=3.0):
    alone = _probe(issue, 0.0)["copy_end_ms"]
    _probe(issue, occupy_ms)  # warm-up (first launches carry setup cost)
    r = _probe(issue, occupy_ms)
    r["alone_ms"] = alone
    return r


def _probe(issue, occupy_ms):
    lib = runtime.load_library()
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s0)
    runtime.check(lib.ficco_occupy_sms(int(occupy_ms * 1e6), C.c_void_p(s0.cuda_stream)))
    e1.record(s0)
    s1.wait_event(e0)
    issue(s1)
    e2.record(s1)
    torch.cuda.synchronize()
    return {"occupy_ms": round(e0.elapsed_time(e1), 3), "copy_end_ms": round(e0.elapsed_time(e2), 3)}


def main():
    rt = cudart()
    n = 56 * MiB
    src = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(3)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    res = {}
    res["memcpy_1d"] = probe(lambda s: rt.cudaMemcpyAsync(C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()),
                                                          C.c_size_t(n), 3, C.c_void_p(s.cuda_stream)))
    res["memcpy_2d"] = probe(lambda s: rt.cudaMemcpy2DAsync(
        C.c_void_p(dst.data_ptr()), C.c_size_t(8192), C.c_void_p(src.data_ptr()), C.c_size_t(16384),
        C.c_size_t(4096), C.c_size_t(n // 16384), 3, C.c_void_p(s.cuda_stream)))

    def batch(s):
        d = (C.c_void_p * 1)(dst.data_ptr())
        sr = (C.c_void_p * 1)(src.data_ptr())
        z = (C.c_size_t * 1)(n)
        runtime.check(runtime.load_library().ficco_copy_batch(d, sr, z, 1, C.c_void_p(s.cuda_stream)))
    res["batch_prefer_overlap"] = probe(batch)
    def tcopy(s):
        with torch.cuda.stream(s):
            dst.copy_(src)
    res["torch_copy"] = probe(tcopy)
    # the AG copy program of a virtual-peer plan (C2 shapes), copies only
    G, R, K, N = 8, 1024, 4096, 3584
    grp = ops.FiccoGroup.virtual_group(G, 0)
    shards = [torch.zeros(R, K, dtype=torch.bfloat16, device="cuda") for _ in range(G)]
    w = torch.zeros(N, K, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(G * R, N, dtype=torch.bfloat16, device="cuda")
    for kind in ("hetero_unfused_1d", "uniform_fused_2d"):
        plan, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, shards)
        res[f"plan_copies_{kind}"] = probe(lambda s: plan.run_parts(shards[0], w, out, s, copies=True, tiles=False))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

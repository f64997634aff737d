"""Decompose the C3 GEMM->RS overhead over the plain GEMM (virtual 8 ranks, hetero_fused_1d).

Variants of the SAME lowered plan, each timed with CUDA events (L2 flushed):
  full          the op as shipped (push copies + STORE_SIGNAL + REDUCE tiles)
  core          comm_agent='core': epilogues store partials straight into the owners' slots
  no_push       push copies dropped (counter waits / virtual flags kept)
  store_only    no copies, every tile a plain STORE (the RS tile ORDER with GEMM epilogues)
  no_reduce     no copies, REDUCE tiles as plain STORE (STORE_SIGNAL kept)
  core_alias    core, but every peer slot read from slot 0 (timing only: partial reads L2-resident)
  core_noadd    core, partial boxes loaded through the ring but no identity MMAs (timing only)
  gemm          ficco_gemm_bf16 of the same M x N x K (row-major tile order)
Usage: python tools/rs_decomp.py [kind] [reps]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import ops, runtime  # noqa: E402
from paper_2512_10236_b200.lowering import lower_rs  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind  # noqa: E402
from paper_2512_10236_b200.runtime import EPI_REDUCE, EPI_STORE, EPI_STORE_SIGNAL, OP_COPY, OP_WAIT_COUNTER  # noqa: E402


def main():
    kind = ScheduleKind(sys.argv[1]) if len(sys.argv) > 1 else ScheduleKind.HETERO_FUSED_1D
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    runtime.load_library()
    G, M, N, K = 8, 16384, 8192, 3584
    R = M // G
    gen = torch.Generator(device="cuda").manual_seed(0)
    a = (torch.rand(M, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=gen, device="cuda") / 60).to(torch.bfloat16)
    out = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
    full_out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    grp = ops.FiccoGroup.virtual_group(G, 0)
    sc = ops._scenario("gemm_rs", M, N, K, G)
    base = lower_rs(sc, kind, 0, virtual=True)
    grp.ensure_workspace(base.ws_bytes)

    def variant(drop_copies, remap):
        low = lower_rs(sc, kind, 0, virtual=True)
        drop = {OP_COPY} if drop_copies else set()
        if EPI_STORE_SIGNAL in remap:  # nobody counts tiles any more: the push chain would wait forever
            drop.add(OP_WAIT_COUNTER)
        o = [op for op in low.ops if op.op not in drop]
        t = list(low.tiles)
        for x in t:
            if x.mode in remap:
                x.mode = remap[x.mode]
                if x.mode == EPI_STORE:  # write own-layout rows: keep it inside the R x N output
                    x.c_row = x.c_row % R
        return runtime.Plan(grp.comm, low.desc, o, t)

    core = lower_rs(sc, kind, 0, virtual=True, comm_agent="core")
    grp.ensure_workspace(max(base.ws_bytes, core.ws_bytes))
    plans = {
        "full": runtime.Plan(grp.comm, base.desc, base.ops, base.tiles),
        "core": runtime.Plan(grp.comm, core.desc, core.ops, core.tiles),
        "no_push": variant(True, {}),
        "no_reduce": variant(True, {EPI_REDUCE: EPI_STORE}),
        "store_only": variant(True, {EPI_REDUCE: EPI_STORE, EPI_STORE_SIGNAL: EPI_STORE}),
    }
    fns = {k: (lambda p=p: p.run(a, w, out)) for k, p in plans.items()}

    def aliased():  # core, every REDUCE reads the peers' partials from slot 0 (wrong sums; L2-resident)
        os.environ["FICCO_RS_ALIAS"] = "1"
        plans["core"].run(a, w, out)
        os.environ.pop("FICCO_RS_ALIAS")
    fns["core_alias"] = aliased

    def no_add():  # core, partials streamed through the ring but not added (wrong sums; timing only)
        os.environ["FICCO_RS_MMA"] = "2"
        plans["core"].run(a, w, out)
        os.environ.pop("FICCO_RS_MMA")
    fns["core_noadd"] = no_add
    fns["gemm"] = lambda: runtime.gemm_bf16(a, w, full_out)
    res = {k: [] for k in fns}
    for _ in range(3):
        for f in fns.values():
            f()
    torch.cuda.synchronize()
    for _ in range(reps):
        for k, f in fns.items():
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            e1.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3)
    grp.comm.check()
    for k, v in res.items():
        print(f"{kind.value:18s} {k:11s} median {statistics.median(v):7.1f} us  min {min(v):7.1f}", flush=True)
    for p in plans.values():
        p.close()
    grp.close()


if __name__ == "__main__":
    main()

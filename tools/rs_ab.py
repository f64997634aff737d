"""Interleaved A/B of GEMM -> RS tile programs (C3 shapes, virtual ranks, ONE group).

Each spec "kind:agent[:ENV=V,ENV=V]" is lowered with those environment settings (lowering-time knobs
such as FICCO_RS_REDUCE_LAG) and run as a raw plan on the same communicator; all variants and the
plain tile GEMM are timed round-robin (L2 flushed before each call), twice.
usage: python tools/rs_ab.py G spec [spec ...]
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import lowering, ops, runtime  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind  # noqa: E402


def main():
    G = int(sys.argv[1])
    specs = []
    for sp in sys.argv[2:]:
        parts = sp.split(":")
        env = dict(kv.split("=") for kv in parts[2].split(",")) if len(parts) > 2 else {}
        specs.append((parts[0], parts[1], env))
    runtime.load_library()
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS["c3"](torch, dev, G, 0, 1, ops)
    grp = ops.FiccoGroup.virtual_group(G, 0)
    for kind, agent, _ in specs:  # size the workspace, load the virtual peers' partials
        wl.agent = agent
        wl.prepare(grp, kind)
    comm0 = grp.comm
    m, n, k = wl.op_shape(G)
    sc = ops._scenario("c3", m, n, k, G)
    variants, plans = [], []
    for kind, agent, env in specs:
        saved = {k_: os.environ.get(k_) for k_ in env}
        os.environ.update(env)
        try:
            low = lowering.lower_rs(sc, ScheduleKind(kind), 0, virtual=True, comm_agent=agent)
        finally:
            for k_, v_ in saved.items():
                if v_ is None:
                    os.environ.pop(k_, None)
                else:
                    os.environ[k_] = v_
        grp.ensure_workspace(low.ws_bytes)
        assert grp.comm is comm0, "workspace grew after the first plan"
        plan = runtime.Plan(grp.comm, low.desc, low.ops, low.tiles)
        plans.append(plan)
        tag = "".join(f",{k_}={v_}" for k_, v_ in env.items())
        variants.append((f"{kind}/{agent}{tag}", (lambda p=plan: p.run(wl.a, wl.w, wl.out))))
    kern_fn, _, _ = wl.kernel(runtime)
    variants.append(("plain tile GEMM", kern_fn))
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    stream = torch.cuda.current_stream()
    res = {}
    for _ in range(2):
        times = bench.time_interleaved([f for _, f in variants], 20, 5, flush, stream)
        for (name, _), ts in zip(variants, times):
            res.setdefault(name, []).append(round(statistics.median(ts) * 1e3, 1))
    grp.comm.check()
    ok = wl.check() if hasattr(wl, "check") else None
    for name, v in res.items():
        print(f"{name:60s} {v}", flush=True)
    print("last variant output parity:", ok)
    for p in plans:
        p.close()
    grp.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"rs_ab_g{G}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

"""Interleaved A/B of the AG copy-program structure (C2 or C4 shapes, virtual 8 ranks, ONE group).

Variants per schedule: full plan; "noflags" (copies run, tiles ignore every gate: copy contention only);
"nocopies" (no copy program, no gates: the tile order alone); fine-grain kinds at several
FICCO_FINE_CHAINS settings. All plans share one communicator (one set of copy streams), and every
variant is timed round-robin with the others (L2 flushed before each call).
usage: python tools/fine_ab.py [c2|c4] [kind ...]
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
from paper_2512_10236_b200.routing import ScheduleKind, build_plan  # noqa: E402

G = 8


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    kinds = sys.argv[2:] or ["shard_overlap_p2p", "hetero_unfused_1d"]
    runtime.load_library()
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS[key](torch, dev, G, 0, 1, ops)
    inplace = key == "c2"
    wl.inplace = inplace
    grp = ops.FiccoGroup.virtual_group(G, 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    m, n, k = wl.op_shape(G)
    sc = ops._scenario(key, m, n, k, G)
    gathered = "B" if key == "c4" else "A"
    variants, plans = [], []
    specs = []
    for kind in kinds:
        if ":" in kind:  # kind:var:chains[:ENV=V,ENV=V] spelled out
            parts = kind.split(":")
            env = dict(kv.split("=") for kv in parts[3].split(",")) if len(parts) > 3 else {}
            specs.append((parts[0], parts[1], parts[2], env))
            continue
        fine = kind not in ("shard_overlap_p2p", "serial")
        for chains in (["0", "4", "2"] if fine else ["0"]):
            for var in (["full", "noflags", "nocopies"] if chains == "0" else ["full"]):
                specs.append((kind, var, chains, {}))
    for kind in sorted({sp[0] for sp in specs}):  # size the workspace, load the virtual peers' shards
        wl.prepare(grp, kind)
    comm0 = grp.comm
    for kind, var, chains, env in specs:
        os.environ["FICCO_FINE_CHAINS"] = chains
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        kw = dict(other_rows=wl.Tq, alpha=wl.scale) if gathered == "B" else {}
        low = lowering.lower_ag(build_plan(sc, ScheduleKind(kind)), 0, gathered, inplace=inplace, **kw)
        for k_, v_ in saved.items():
            if v_ is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v_
        grp.ensure_workspace(low.ws_bytes)
        assert grp.comm is comm0, "workspace grew after the first plan"
        if var == "nosignal":  # tiles ignore gates AND the copy program writes no flags
            low.ops = [o for o in low.ops if o.op != runtime.OP_SIGNAL]
        if var in ("noflags", "nocopies", "nosignal"):
            for t in low.tiles:
                t.flag, t.fmask = -1, 0
        if var == "nocopies":
            low.ops = []
        plan = runtime.Plan(grp.comm, low.desc, low.ops, low.tiles)
        plans.append(plan)
        tag = "".join(f",{k_}={v_}" for k_, v_ in env.items())
        variants.append((f"{kind}/{var}/chains={chains}{tag}", (lambda p=plan: wl.run_plan(p))))
    os.environ.pop("FICCO_FINE_CHAINS", None)
    kern_fn, _, _ = wl.kernel(runtime)
    variants.append(("plain tile GEMM", kern_fn))
    stream = torch.cuda.current_stream()
    res = {}
    for rep in range(2):
        times = bench.time_interleaved([f for _, f in variants], 25, 5, flush, stream)
        for (name, _), ts in zip(variants, times):
            res.setdefault(name, []).append(round(statistics.median(ts) * 1e3, 1))
    grp.comm.check()
    for name, v in res.items():
        print(f"{name:70s} {v}", flush=True)
    for p in plans:
        p.close()
    grp.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"fine_ab_{key}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

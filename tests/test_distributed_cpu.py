"""N > 1 host path with real processes on CPU (gloo, world_size 2).

Each process plays one rank: it exchanges its (fake) workspace handle through
torch.distributed exactly like Communicator.from_process_group, lowers its own
copy/tile programs for every schedule, and ships them to rank 0, which executes
both ranks' programs with the multi-rank interpreter and checks the outputs.
"""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

KINDS = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d",
         "uniform_fused_2d"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _to_plain(low):
    """ctypes programs -> picklable tuples (and back in rank 0)."""
    ops = [{f: getattr(o, f) for f, _ in type(o)._fields_} for o in low.ops]
    tiles = [{f: getattr(t, f) for f, _ in type(t)._fields_} for t in low.tiles]
    d = low.desc
    desc = {f: (getattr(d, f) if not hasattr(getattr(d, f), "_fields_")
                else {g: getattr(getattr(d, f), g) for g, _ in type(getattr(d, f))._fields_})
            for f, _ in type(d)._fields_ if f not in ("ops", "tiles")}
    return {"ops": ops, "tiles": tiles, "desc": desc, "ws_bytes": low.ws_bytes,
            "gather_off": low.gather_off, "gather_par": low.gather_par}


def _from_plain(doc):
    from paper_2512_10236_b200 import runtime
    from paper_2512_10236_b200.lowering import Lowered
    low = Lowered()
    low.ops = [runtime.CopyOp(**o) for o in doc["ops"]]
    low.tiles = [runtime.Tile(**t) for t in doc["tiles"]]
    for f, v in doc["desc"].items():
        if isinstance(v, dict):
            setattr(low.desc, f, runtime.Operand(**v))
        else:
            setattr(low.desc, f, v)
    low.ws_bytes, low.gather_off, low.gather_par = doc["ws_bytes"], doc["gather_off"], doc["gather_par"]
    return low


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_10236_b200 import runtime
        from paper_2512_10236_b200.lowering import lower_ag
        from paper_2512_10236_b200.ops import _scenario
        from paper_2512_10236_b200.routing import ScheduleKind, build_plan
        handles = runtime.exchange_handles(bytes([rank]) * 64)
        assert [h[0] for h in handles] == list(range(world))
        progs = {}
        sc = _scenario("dist", 64 * world, 64, 256, world)
        for kind in KINDS:
            progs[kind] = _to_plain(lower_ag(build_plan(sc, ScheduleKind(kind)), rank, "A"))
        gathered = [None] * world
        dist.all_gather_object(gathered, pickle.dumps(progs))
        if rank == 0:
            q.put(gathered)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_process_lowering_and_protocol():
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle import ficco_oracle as orc
    from protocol_sim import World, bf16_bits, bits_f32
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    per_rank = [pickle.loads(g) for g in gathered]
    R, K, N = 64, 256, 64
    for kind in KINDS:
        lows = [_from_plain(per_rank[r][kind]) for r in range(world)]
        w = orc.seeded_inputs(3, 99, (N, K), "normal")
        args, expect = [], []
        for run in range(3):
            shards = [orc.seeded_inputs(run, g, (R, K)) for g in range(world)]
            expect.append(np.concatenate(shards) @ w.T)
            args.append([{"a": bf16_bits(shards[g]), "b": bf16_bits(w),
                          "c": np.zeros((R * world, N), dtype=np.uint16)} for g in range(world)])
        sim = World(lows, args, seed=1)
        sim.on_run_done = lambda rank, run: np.testing.assert_allclose(
            bits_f32(args[run][rank]["c"]), expect[run], rtol=2e-2, atol=2e-2)
        sim.run(3)

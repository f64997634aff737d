"""Real executor twin of the reference's ``engine.simulate`` (engine.py:117).

``execute(plan, ...)`` runs one rank's share of an ``ExecutionPlan`` on the
B200 (copy engines + tcgen05 tile kernel through the C-ABI) and returns the
outputs together with a ``SimResult`` in the simulator's schema built from the
measurement:

* ``makespan`` — CUDA-event time of the whole op on the compute stream;
* ``timeline`` — one ``TaskSpan`` per GemmSpec task of this rank (first tile
  load start -> last tile stored, from the kernel's %globaltimer trace) and per
  arriving TransferSpec (start = kernel start; end = when the first tile gated
  on its readiness flag started loading, an upper bound on the arrival), so
  measured and simulated runs diff with ``export_trace_csv`` (engine.py:310-318).

``measured_makespan(kind_scenario)`` is the ``makespan_fn`` hook of
``selector.validate_heuristic``: exhaustive search over measured makespans
instead of the analytic model.
"""

from __future__ import annotations

import statistics

import torch

from . import ops
from .lowering import F_RING, F_XFER, lower_ag
from .routing import ExecutionPlan, GemmSpec, ScheduleKind, TransferSpec, build_plan
from .simulator import SimResult, TaskSpan


def _gemm_tile_groups(plan: ExecutionPlan, rank: int, low) -> list[tuple[int, list[int]]]:
    """(task id, tile indices) per GemmSpec of this rank, matched by output rows."""
    tiles = low.tiles
    groups = []
    for t in plan.tasks:
        if t.gpu != rank or not isinstance(t.kind, GemmSpec):
            continue
        if t.kind.col_block is not None:
            if t.kind.col_block[0] != 0:
                continue
            idx = [i for i, tl in enumerate(tiles) if tl.rows > 0]
        else:
            idx = [i for i, tl in enumerate(tiles)
                   if tl.rows > 0 and any(s <= tl.c_row < s + c for s, c in t.kind.rows)]
        groups.append((t.id, idx))
    return groups


def _first_gate(tile) -> list[int]:
    """Readiness flags a tile waits for before its first k-block (segment 0 for k-segmented tiles)."""
    return [tile.flag + b for b in range(16) if tile.fmask >> b & 1]


def _transfer_flag(plan: ExecutionPlan, x: TransferSpec, rank: int) -> int:
    """The flag the lowered copy program sets when transfer ``x`` has landed (lowering.lower_ag)."""
    G = plan.scenario.n_gpus
    if plan.schedule is ScheduleKind.SHARD_OVERLAP_P2P:
        return F_RING + x.round_idx + 1
    return F_XFER + x.round_idx * G + x.src


def execute(plan: ExecutionPlan, a_shard: torch.Tensor, weight: torch.Tensor, group: "ops.FiccoGroup",
            out: torch.Tensor | None = None, warmup: int = 2) -> tuple[torch.Tensor, SimResult]:
    """Run an all-gather -> GEMM plan for this rank; returns (C, measured SimResult)."""
    if plan.schedule is ScheduleKind.IDEAL:
        raise ValueError("ideal is a pricing bound, not an executable schedule")
    rank = group.rank
    sc = plan.scenario
    key = ("exec", sc.gemm.m, sc.gemm.n, sc.gemm.k, plan.schedule)
    pl, low = group.plan(key, lambda: lower_ag(plan, rank, "A"))
    if out is None:
        out = torch.empty(sc.gemm.m, sc.gemm.n, dtype=torch.bfloat16, device=a_shard.device)
    info = pl.info()
    trace = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device=a_shard.device)
    pl.set_trace(trace)
    try:
        for _ in range(warmup):
            pl.run(a_shard, weight, out)
        times = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            pl.run(a_shard, weight, out)
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e) * 1e-3)
        group.comm.check()
    finally:
        tr = trace.cpu().tolist()
        pl.set_trace(None)
    grid = info["grid"]
    t0 = min(tr[:grid])
    ready = [(tr[grid + 2 * i] - t0) * 1e-9 for i in range(info["tiles"])]
    done = [(tr[grid + 2 * i + 1] - t0) * 1e-9 for i in range(info["tiles"])]
    spans = []
    for tid, idx in _gemm_tile_groups(plan, rank, low):
        if idx:
            spans.append(TaskSpan(tid, rank, "gemm", min(ready[i] for i in idx), max(done[i] for i in idx), 0.0))
    # a transfer has landed no later than the first tile gated on its readiness flag started
    # its loads (the tile producer's stamp is taken right after its first gate is satisfied)
    first_gated: dict[int, float] = {}
    for i, tl in enumerate(low.tiles):
        if tl.rows > 0 and tl.flag >= 0:
            for f in _first_gate(tl):
                first_gated[f] = min(first_gated.get(f, ready[i]), ready[i])
    for t in plan.tasks:
        if isinstance(t.kind, TransferSpec) and t.kind.dst == rank:
            end = first_gated.get(_transfer_flag(plan, t.kind, rank))
            if end is not None:
                spans.append(TaskSpan(t.id, rank, f"transfer[{t.kind.src}->{t.kind.dst}]", 0.0, end, 0.0))
    spans.sort(key=lambda s: s.task_id)
    res = SimResult(sc.name, plan.schedule, statistics.median(times), tuple(spans), {}, 0.0)
    return out, res


class MeasuredMakespan:
    """``makespan_fn`` for ``validate_heuristic``: measured seconds per plan (rank 0, virtual peers)."""

    def __init__(self, warmup: int = 3, reps: int = 10):
        self.warmup, self.reps = warmup, reps
        self.cache: dict = {}

    def __call__(self, plan: ExecutionPlan) -> float:
        sc = plan.scenario
        key = (sc.gemm.m, sc.gemm.n, sc.gemm.k, sc.n_gpus, plan.schedule)
        if key in self.cache:
            return self.cache[key]
        G, R, K, N = sc.n_gpus, sc.gemm.m // sc.n_gpus, sc.gemm.k, sc.gemm.n
        grp = ops.FiccoGroup.virtual_group(G, 0)
        try:
            gen = torch.Generator(device="cuda").manual_seed(0)
            shards = [(torch.rand(R, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(G)]
            w = (torch.randn(N, K, generator=gen, device="cuda") / K ** 0.5).to(torch.bfloat16)
            out = torch.empty(sc.gemm.m, N, dtype=torch.bfloat16, device="cuda")
            kind = plan.schedule
            _, low, _ = ops.prepare_ag(grp, R, K, N, kind)
            grp.load_peer_shards(low, shards)
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            for _ in range(self.warmup):
                ops.all_gather_matmul(shards[0], w, kind=kind, group=grp, out=out)
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(self.reps)]
            torch.cuda._sleep(100_000_000)  # host enqueues every rep before the GPU gets there
            for s, e in evs:
                flush.fill_(1)  # L2 flushed between reps
                s.record()
                ops.all_gather_matmul(shards[0], w, kind=kind, group=grp, out=out)
                e.record()
            torch.cuda.synchronize()
            ts = [s.elapsed_time(e) * 1e-3 for s, e in evs]
            grp.comm.check()
        finally:
            grp.close()
        self.cache[key] = statistics.median(ts)
        return self.cache[key]


__all__ = ["execute", "MeasuredMakespan", "build_plan"]

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
from .lowering import F_RING, F_XFER
from .routing import ExecutionPlan, GemmSpec, ScheduleKind, TransferSpec, build_plan
from .simulator import SimResult, TaskSpan


def _gemm_tile_groups(plan: ExecutionPlan, rank: int, low, gathered: str = "A") -> list[tuple[int, list[int]]]:
    """(task id, tile indices) per GemmSpec of this rank, matched by the plan rows a tile computes
    (output rows for the gathered-A ops; output COLUMNS for the CP gathered-B op, whose plan rows are
    kv tokens)."""
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
            pos = (lambda tl: tl.c_col) if gathered == "B" else (lambda tl: tl.c_row)
            idx = [i for i, tl in enumerate(tiles)
                   if tl.rows > 0 and any(s <= pos(tl) < s + c for s, c in t.kind.rows)]
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


def _timed_runs(pl, run, warmup: int, reps: int = 3) -> tuple[list[float], list[int], dict]:
    """Run ``run()`` (one op through plan ``pl``) warmup + reps times with the kernel trace attached;
    returns (seconds per rep, the last rep's trace, plan info)."""
    info = pl.info()
    trace = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device="cuda")
    pl.set_trace(trace)
    try:
        for _ in range(warmup):
            run()
        times = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run()
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e) * 1e-3)
    finally:
        tr = trace.cpu().tolist()
        pl.set_trace(None)
    return times, tr, info


def execute(plan: ExecutionPlan, a: torch.Tensor, weight: torch.Tensor, group: "ops.FiccoGroup",
            out: torch.Tensor | None = None, warmup: int = 2, op: str = "ag", comm_agent: str = "dma",
            scale: float | None = None) -> tuple[torch.Tensor, SimResult]:
    """Run one rank's share of ``plan`` on the B200 and return (output, measured SimResult).

    op 'ag'  all-gather -> GEMM: a = A shard [R, K], weight [N, K] (plan = the AG scenario);
    op 'a2a' all-to-all -> expert GEMM: a = send buffer [M, K] (plan of an all_to_all scenario);
    op 'cp'  CP KV all-gather -> QK^T: a = Q [Tq, d], weight = K shard [Tkv/G, d] (plan scenario
             (M, N, K) = (Tkv, Tq, d));
    op 'rs'  GEMM -> reduce-scatter: a = A [M, Kg], weight [N, Kg] (plan = the schedule kind's AG plan
             of the same scenario; the executed program is its adjoint, lowering.rs_pieces).
    The timeline is in the simulator's schema (export_trace_csv, engine.py:310-318): one span per
    GemmSpec task (first tile load start -> last tile stored; RS: per pushed piece / own reduce piece)
    and per arriving transfer (AG/A2A/CP: kernel start -> first tile gated on its flag started).
    """
    if plan.schedule is ScheduleKind.IDEAL:
        raise ValueError("ideal is a pricing bound, not an executable schedule")
    if op not in ("ag", "a2a", "cp", "rs"):
        raise ValueError(f"op must be 'ag', 'a2a', 'cp' or 'rs', got {op!r}")
    rank, sc, kind = group.rank, plan.scenario, plan.schedule
    M, N, K = sc.gemm.m, sc.gemm.n, sc.gemm.k
    G = sc.n_gpus
    if op == "rs":
        pl, low, _ = ops.prepare_rs(group, M, K, N, kind, comm_agent=comm_agent)
        shape, run_op = (M // G, N), "gemm_rs"
    elif op == "cp":
        pl, low, _ = ops.prepare_cp(group, N, K, M, kind, scale, comm_agent=comm_agent)
        shape, run_op = (N, M), "cp_qk"
    elif op == "a2a":
        pl, low, _ = ops.prepare_a2a(group, M // G, K, N, kind, comm_agent=comm_agent)
        shape, run_op = (M, N), "a2a_gemm"
    else:
        pl, low, _ = ops.prepare_ag(group, M // G, K, N, kind, comm_agent=comm_agent)
        shape, run_op = (M, N), "ag_gemm"
    if out is None:
        out = torch.empty(*shape, dtype=torch.bfloat16, device=a.device)
    times, tr, info = _timed_runs(pl, lambda: pl.run_op(run_op, a, weight, out), warmup)
    group.comm.check()
    grid = info["grid"]
    t0 = min(tr[:grid])
    ready = [(tr[grid + 2 * i] - t0) * 1e-9 for i in range(info["tiles"])]
    done = [(tr[grid + 2 * i + 1] - t0) * 1e-9 for i in range(info["tiles"])]
    spans = []
    if op == "rs":
        spans = _rs_spans(sc, kind, rank, low, ready, done)
    else:
        for tid, idx in _gemm_tile_groups(plan, rank, low, "B" if op == "cp" else "A"):
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
    res = SimResult(sc.name, kind, statistics.median(times), tuple(spans), {}, 0.0)
    return out, res


def _rs_spans(sc, kind, rank, low, ready, done) -> list[TaskSpan]:
    """GEMM -> RS timeline: one span per piece of the schedule's adjoint routing (lowering.rs_pieces), in
    emission order: 'gemm[->q]' for a remote owner's partial (its push starts when the span ends),
    'reduce' for the own rows folded with the received partials. Task ids number the pieces."""
    from .lowering import EPI_REDUCE, EPI_STORE_REMOTE, rs_pieces
    order, _ = rs_pieces(sc, kind, rank)
    R = sc.gemm.m // sc.n_gpus
    spans = []
    for pid, (remote, pc) in enumerate(order):
        idx = []
        for i, tl in enumerate(low.tiles):
            if tl.rows <= 0 or (tl.mode == EPI_REDUCE) == remote:
                continue
            row = tl.c_row + (tl.chunk * R if tl.mode == EPI_STORE_REMOTE else 0) if remote else tl.c_row + rank * R
            if pc.row0 <= row < pc.row0 + pc.nrows and pc.col0 <= tl.c_col < pc.col0 + pc.ncols:
                idx.append(i)
        if idx:
            spans.append(TaskSpan(pid, rank, f"gemm[->{pc.owner}]" if remote else "reduce",
                                  min(ready[i] for i in idx), max(done[i] for i in idx), 0.0))
    return spans


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

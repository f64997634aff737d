"""Lower an ExecutionPlan (one rank's share) into the executor's copy + tile programs.

The reference DAG (planner.py:58-113) is executed on B200 as:

* every ``TransferSpec`` arriving at this rank -> a copy-engine COPY that
  *pulls* the chunk from the source rank's symmetric workspace straight into
  its final row offset of the local gathered buffer, followed (per the kind's
  dependency granularity) by a SIGNAL of a readiness flag;
* every ``GemmSpec`` -> the 128x256 output tiles of its row fragments
  (``rows``) or its K block (``col_block``), in plan order, each gated by the
  flag covering the rows it reads;
* ``GatherSpec`` / ``ScatterSpec`` -> nothing (folded into copy destinations
  and epilogue addressing).

Schedule kinds therefore differ only in tile order and dependency sets
(SURVEY.md §7 step 4):

=================  ===================================  =====================================
kind               copy program (rank g)                tile order / gating
=================  ===================================  =====================================
serial             all G-1 shards, one flag ALL          whole GEMM gated on ALL
shard_overlap_p2p  ring: step i pulls shard (g-i)%G      shard-major; step i gated on RING[i]
                   from the left neighbour, who
                   notifies when it holds it
uniform_fused_1d   round c: chunk c of every peer,       step s: chunk s of every shard
                   flag ROUND[c]                          (local rows gated on LOCAL)
hetero_fused_1d    same as uniform                       local shard first, then per round
hetero_unfused_1d  per (round, peer) flag XFER[c,p]      per (round, peer) chunk GEMMs
uniform_fused_2d   round c: R x b slab of every peer     output-stationary; k-block kb of a
                   (2D CE copy), flag ROUND[c]           peer's rows gated on ROUND[kb/kseg]
=================  ===================================  =====================================

Every plan starts with a publish barrier (each rank copies its shard into its
own slot, notifies PUB to all peers and waits for theirs) which, with the
epoch-parity double buffer, makes back-to-back calls race-free.

GEMM -> reduce-scatter (R1) and context-parallel QK^T (R2) are not in the
reference; they are lowered here as the adjoint and the
transposed-operand variants of the same chunk routing (see ``lower_rs`` /
``lower_ag(..., gathered="B")``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .domain import Scenario
from .routing import (ExecutionPlan, GatherSpec, GemmSpec, PlanError, ScatterSpec, ScheduleKind, TransferSpec,
                      build_plan)
from .runtime import (BUF_A, BUF_B, BUF_C, BUF_NONE, BUF_WS, EPI_REDUCE, EPI_STORE, EPI_STORE_SIGNAL,
                      FICCO_FLAG_COUNTERS, FICCO_WS_DATA_OFFSET, MAX_RECV, OP_COPY, OP_NOTIFY, OP_SIGNAL,
                      OP_WAIT, OP_WAIT_COUNTER, TILE_K, TILE_M, TILE_N, CopyOp, Operand, PlanDesc, Tile)

# flag word map (local flag area of each rank's workspace)
F_PUB = 0        # + src rank: "src has published this epoch's shard"
F_LOCAL = 64     # local shard copied into its own slot
F_ROUND = 65     # + round c: all chunks of round c landed
F_XFER = 256     # + c*G + p: chunk (p, c) landed (unfused)
F_RING = 512     # + step i: ring step i landed
F_RINGN = 576    # + step i: left neighbour holds the shard we pull at step i+1
F_ALL = 640      # serial: every shard landed
F_DONE = 704     # + src rank: "src finished its previous run" (RS receive-buffer reuse)
F_RS = 1024      # + chunk*(G-1) + slot: partial chunk from a peer landed (RS)

ELT = 2  # bf16


@dataclass
class Lowered:
    """A rank's program, ready for ``runtime.Plan``."""

    ops: list[CopyOp] = field(default_factory=list)
    tiles: list[Tile] = field(default_factory=list)
    desc: PlanDesc = field(default_factory=PlanDesc)
    ws_bytes: int = FICCO_WS_DATA_OFFSET
    gather_off: int = 0      # byte offset of parity-0 gathered buffer in the workspace
    gather_par: int = 0      # parity stride
    recv_off: int = 0
    recv_par: int = 0
    recv_slot: int = 0
    notes: dict = field(default_factory=dict)


def _op(op, **kw) -> CopyOp:
    c = CopyOp()
    c.op = op
    c.peer = kw.pop("peer", -1)
    c.flag = kw.pop("flag", 0)
    c.dst_peer = kw.pop("dst_peer", -1)
    c.height = kw.pop("height", 1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _operand(buf, rows, ld, off=0, par=0) -> Operand:
    o = Operand()
    o.buf, o.off, o.par, o.rows, o.ld = buf, off, par, rows, ld
    return o


def _tile(a_row, b_row, c_row, c_col, rows, cols, flag=-1, kseg=0, mode=EPI_STORE, chunk=0, recv_row=0) -> Tile:
    t = Tile()
    t.a_row, t.b_row, t.c_row, t.c_col = a_row, b_row, c_row, c_col
    t.rows, t.cols, t.flag, t.kseg, t.mode, t.chunk, t.recv_row = rows, cols, flag, kseg, mode, chunk, recv_row
    return t


def _check_shape(m: int, n: int, k: int) -> None:
    if k % 8:
        raise PlanError(f"K={k} must be a multiple of 8 (16-byte TMA rows)")
    if n % 32:
        raise PlanError(f"N={n} must be a multiple of 32 (epilogue column granularity)")


def _my_gemms(plan: ExecutionPlan, rank: int) -> list[GemmSpec]:
    return [t.kind for t in plan.tasks if t.gpu == rank and isinstance(t.kind, GemmSpec)]


def _publish(ops: list, g: int, world: int, row_bytes: int, shard_rows: int, gather_off: int, par: int,
             src_buf: int) -> None:
    """Local shard -> own slot, then the cross-rank publish barrier."""
    ops.append(_op(OP_COPY, src_buf=src_buf, dst_buf=BUF_WS, src_off=0, dst_off=gather_off + g * shard_rows * row_bytes,
                   dst_par=par, width=shard_rows * row_bytes))
    ops.append(_op(OP_SIGNAL, flag=F_LOCAL))
    for p in range(world):
        if p != g:
            ops.append(_op(OP_NOTIFY, peer=p, flag=F_PUB + g))
    for p in range(world):
        if p != g:
            ops.append(_op(OP_WAIT, flag=F_PUB + p))


def lower_ag(plan: ExecutionPlan, rank: int, gathered: str = "A", alpha: float = 1.0, grid: int = 0,
             other_rows: int | None = None) -> Lowered:
    """All-gather -> GEMM family (AG->GEMM and the CP KV-gather -> QK^T).

    gathered="A": C[M,N] = A_all[M,K] @ W[N,K]^T; call args (a=A_shard[R,K], b=W, c=C).
    gathered="B": S[Q,M] = alpha * Q[Q,K] @ K_all[M,K]^T; call args (a=Q, b=K_shard[R,K], c=S);
                  the plan's M rows (kv tokens) become output columns; ``other_rows`` = Q.
    """
    sc = plan.scenario
    kind = plan.schedule
    g, G = rank, sc.n_gpus
    M, N, K = sc.gemm.m, sc.gemm.n, sc.gemm.k
    if sc.gemm.elt_bytes != ELT:
        raise PlanError("the B200 executor computes in bf16 (elt_bytes=2)")
    if kind is ScheduleKind.IDEAL:
        raise PlanError("ideal is the loss-free pricing bound, not an executable schedule")
    if gathered not in ("A", "B"):
        raise ValueError("gathered must be 'A' or 'B'")
    _check_shape(M, N, K)
    R = M // G
    row_bytes = K * ELT
    low = Lowered()
    low.gather_off = FICCO_WS_DATA_OFFSET
    low.gather_par = M * row_bytes
    low.ws_bytes = FICCO_WS_DATA_OFFSET + 2 * low.gather_par
    ops = low.ops
    src_buf = BUF_A if gathered == "A" else BUF_B
    _publish(ops, g, G, row_bytes, R, low.gather_off, low.gather_par, src_buf)

    def pull(p: int, row0: int, nrows: int) -> CopyOp:
        off = low.gather_off + row0 * row_bytes
        return _op(OP_COPY, peer=p, src_buf=BUF_WS, dst_buf=BUF_WS, src_off=off, dst_off=off,
                   src_par=low.gather_par, dst_par=low.gather_par, width=nrows * row_bytes)

    # ---- copy program (mirrors the plan's TransferSpecs arriving at this rank)
    xfers = [t.kind for t in plan.tasks if isinstance(t.kind, TransferSpec) and t.kind.dst == g]
    kseg = 0
    if kind is ScheduleKind.SERIAL:
        for x in xfers:
            ops.append(pull(x.src, x.src * R, R))
        ops.append(_op(OP_SIGNAL, flag=F_ALL))
    elif kind is ScheduleKind.SHARD_OVERLAP_P2P:
        right = (g + 1) % G
        if G > 1:
            ops.append(_op(OP_NOTIFY, peer=right, flag=F_RINGN + 0))
        for x in xfers:  # step i = round_idx + 1, from the left neighbour
            i = x.round_idx + 1
            shard = (g - i) % G
            ops.append(_op(OP_WAIT, flag=F_RINGN + i - 1))
            ops.append(pull(x.src, shard * R, R))
            ops.append(_op(OP_SIGNAL, flag=F_RING + i))
            if i < G - 1:
                ops.append(_op(OP_NOTIFY, peer=right, flag=F_RINGN + i))
    elif kind is ScheduleKind.UNIFORM_FUSED_2D:
        b = K // G
        if b % TILE_K:
            raise PlanError(f"uniform_fused_2d on B200 needs K/G={b} to be a multiple of {TILE_K}")
        kseg = b // TILE_K
        last_round = None
        for x in xfers:
            if last_round is not None and x.round_idx != last_round:
                ops.append(_op(OP_SIGNAL, flag=F_ROUND + last_round))
            c = x.round_idx
            off = low.gather_off + x.src * R * row_bytes + c * b * ELT
            ops.append(_op(OP_COPY, peer=x.src, src_buf=BUF_WS, dst_buf=BUF_WS, src_off=off, dst_off=off,
                           src_par=low.gather_par, dst_par=low.gather_par, width=b * ELT, height=R,
                           src_pitch=row_bytes, dst_pitch=row_bytes))
            last_round = c
        if last_round is not None:
            ops.append(_op(OP_SIGNAL, flag=F_ROUND + last_round))
    else:  # the three 1D fine-grain kinds
        r = M // (G * G)
        unfused = kind is ScheduleKind.HETERO_UNFUSED_1D
        last_round = None
        for x in xfers:
            c = x.round_idx
            if not unfused and last_round is not None and c != last_round:
                ops.append(_op(OP_SIGNAL, flag=F_ROUND + last_round))
            ops.append(pull(x.src, x.src * R + c * r, r))
            if unfused:
                ops.append(_op(OP_SIGNAL, flag=F_XFER + c * G + x.src))
            last_round = c
        if not unfused and last_round is not None:
            ops.append(_op(OP_SIGNAL, flag=F_ROUND + last_round))

    # ---- tile program (mirrors this rank's GemmSpecs in plan order)
    def rows_flag(start: int) -> int:
        owner = start // R
        if owner == g:
            return F_LOCAL
        if kind is ScheduleKind.SERIAL:
            return F_ALL
        if kind is ScheduleKind.SHARD_OVERLAP_P2P:
            return F_RING + (g - owner) % G
        c = (start - owner * R) // (M // (G * G))
        if kind is ScheduleKind.HETERO_UNFUSED_1D:
            return F_XFER + c * G + owner
        return F_ROUND + c

    Q = other_rows if gathered == "B" else None
    if gathered == "B" and Q is None:
        raise ValueError("gathered='B' needs other_rows (query rows)")
    tiles = low.tiles
    for spec in _my_gemms(plan, g):
        if spec.col_block is not None:  # uniform_fused_2d: one output-stationary pass over all K
            if spec.col_block[0] != 0:
                continue  # later K blocks accumulate in TMEM inside the same tiles
            frags = [(p * R, R) for p in range(G)]
        else:
            frags = []
            for start, count in spec.rows:  # split at shard boundaries: each piece has one owner/flag
                end = start + count
                while start < end:
                    stop = min(end, (start // R + 1) * R)
                    frags.append((start, stop - start))
                    start = stop
        for start, count in frags:
            owner = start // R
            if kind is ScheduleKind.UNIFORM_FUSED_2D:
                flag, ks = (F_LOCAL, 0) if owner == g else (F_ROUND, kseg)
            else:
                flag, ks = rows_flag(start), 0
            # split the fragment so that no tile straddles an owner (flag) boundary
            if gathered == "A":
                for m0 in range(start, start + count, TILE_M):
                    rows = min(TILE_M, start + count - m0)
                    for n0 in range(0, N, TILE_N):
                        tiles.append(_tile(m0, n0, m0, n0, rows, min(TILE_N, N - n0), flag, ks))
            else:
                if count % 32:
                    raise PlanError(f"gathered-B fragments must be multiples of 32 rows, got {count}")
                for n0 in range(start, start + count, TILE_N):
                    cols = min(TILE_N, start + count - n0)
                    for m0 in range(0, Q, TILE_M):
                        tiles.append(_tile(m0, n0, m0, n0, min(TILE_M, Q - m0), cols, flag, ks))

    d = low.desc
    gat = _operand(BUF_WS, M, K, low.gather_off, low.gather_par)
    if gathered == "A":
        d.a, d.b, d.c = gat, _operand(BUF_B, N, K), _operand(BUF_C, M, N)
    else:
        d.a, d.b, d.c = _operand(BUF_A, Q, K), gat, _operand(BUF_C, Q, M)
    d.part = _operand(BUF_NONE, 0, 0)
    d.recv = _operand(BUF_NONE, 0, 0)
    d.k, d.alpha, d.grid = K, alpha, grid
    low.notes = {"kind": kind.value, "rank": g, "world": G, "gathered": gathered}
    return low


def rs_plan(scenario: Scenario, kind: ScheduleKind) -> ExecutionPlan:
    """The AG plan whose routing the RS schedule is the adjoint of (same chunks, reversed flow)."""
    if kind not in (ScheduleKind.UNIFORM_FUSED_1D, ScheduleKind.HETERO_FUSED_1D, ScheduleKind.HETERO_UNFUSED_1D):
        raise PlanError(f"GEMM->reduce-scatter supports the 1D fine-grain kinds, not {kind.value}")
    return build_plan(scenario, kind)


def lower_rs(scenario: Scenario, kind: ScheduleKind, rank: int, grid: int = 0) -> Lowered:
    """GEMM -> reduce-scatter (not in the reference, parity unpinned).

    Rank g holds A_g [M, Kg] and W_g [N, Kg]; P_g = A_g @ W_g^T [M, N]; rank q
    ends with C_q = sum_g P_g[q*R:(q+1)*R] [R, N]. Fine chunk (q, c) = rows
    q*R + c*r. Partial tiles of remote chunks are stored to the local partial
    buffer and counted; the copy stream pushes each finished chunk into the
    owner's receive slot (copy engine) and notifies it; the owner's tiles of
    its own chunk reduce ``acc + sum_j recv_j`` in the epilogue
    (rank-ascending over the G-1 peers, fp32, one bf16 rounding).

    uniform_fused_1d: round c = remote chunks c (rotated owners) then own chunk c.
    hetero_fused_1d:  all remote chunks round by round, own shard last; push per round.
    hetero_unfused_1d: as fused but each chunk is pushed as soon as it is done.
    """
    plan = rs_plan(scenario, kind)  # validates divisibility exactly like the AG schedule
    g, G = rank, scenario.n_gpus
    M, N, K = scenario.gemm.m, scenario.gemm.n, scenario.gemm.k
    _check_shape(M, N, K)
    if G - 1 > MAX_RECV:
        raise PlanError(f"at most {MAX_RECV + 1} ranks")
    R, r = M // G, M // (G * G)
    row_bytes = N * ELT
    low = Lowered()
    part_off = FICCO_WS_DATA_OFFSET
    low.recv_off = part_off + M * row_bytes
    low.recv_slot = R * row_bytes
    low.recv_par = (G - 1) * low.recv_slot
    low.ws_bytes = low.recv_off + 2 * low.recv_par
    ops, tiles = low.ops, low.tiles
    unfused = kind is ScheduleKind.HETERO_UNFUSED_1D

    def slot_of(src: int, owner: int) -> int:
        return src if src < owner else src - 1

    # units of work that are pushed together: list of (counter id, [(owner q, round c)])
    units: list[tuple[int, list[tuple[int, int]]]] = []
    order: list[tuple[str, int, int]] = []  # ("remote"|"own", q, c) tile emission order
    for c in range(G):
        remote = [((g + j) % G, c) for j in range(1, G)]
        if unfused:
            for q, cc in remote:
                units.append((len(units), [(q, cc)]))
        else:
            units.append((len(units), remote))
        order += [("remote", q, cc) for q, cc in remote]
        if kind is ScheduleKind.UNIFORM_FUSED_1D:
            order.append(("own", g, c))
    if kind is not ScheduleKind.UNIFORM_FUSED_1D:
        order += [("own", g, c) for c in range(G)]
    unit_of = {qc: uid for uid, qcs in units for qc in qcs}

    tiles_per_chunk = ((r + TILE_M - 1) // TILE_M) * ((N + TILE_N - 1) // TILE_N)
    for what, q, c in order:
        row0 = q * R + c * r
        for m0 in range(row0, row0 + r, TILE_M):
            rows = min(TILE_M, row0 + r - m0)
            for n0 in range(0, N, TILE_N):
                cols = min(TILE_N, N - n0)
                if what == "remote":
                    tiles.append(_tile(m0, n0, m0, n0, rows, cols, mode=EPI_STORE_SIGNAL, chunk=unit_of[(q, c)]))
                else:
                    local = m0 - g * R
                    tiles.append(_tile(m0, n0, local, n0, rows, cols, mode=EPI_REDUCE, chunk=c, recv_row=local))

    # copy program
    for p in range(G):
        if p != g:
            ops.append(_op(OP_NOTIFY, peer=p, flag=F_DONE + g))
    waited_done: set[int] = set()
    for uid, qcs in units:
        ops.append(_op(OP_WAIT_COUNTER, flag=uid, value=tiles_per_chunk * len(qcs)))
        for q, c in qcs:
            if q not in waited_done:
                ops.append(_op(OP_WAIT, flag=F_DONE + q, value=1))
                waited_done.add(q)
            src = part_off + (q * R + c * r) * row_bytes
            dst = low.recv_off + slot_of(g, q) * low.recv_slot + c * r * row_bytes
            ops.append(_op(OP_COPY, src_buf=BUF_WS, dst_buf=BUF_WS, dst_peer=q, src_off=src, dst_off=dst,
                           dst_par=low.recv_par, width=r * row_bytes))
        for q, c in qcs:
            ops.append(_op(OP_NOTIFY, peer=q, flag=F_RS + c * (G - 1) + slot_of(g, q)))

    d = low.desc
    d.a, d.b = _operand(BUF_A, M, K), _operand(BUF_B, N, K)
    d.c = _operand(BUF_C, R, N)
    d.part = _operand(BUF_WS, M, N, part_off)
    d.recv = _operand(BUF_WS, R, N, low.recv_off, low.recv_par)
    d.recv_slot, d.n_recv, d.rs_flag0 = low.recv_slot, G - 1, F_RS
    d.n_counters = len(units)
    d.k, d.alpha, d.grid = K, 1.0, grid
    if len(units) >= 4096 - 1:
        raise PlanError("too many push units")
    low.notes = {"kind": kind.value, "rank": g, "world": G, "op": "rs", "units": len(units),
                 "tiles_per_chunk": tiles_per_chunk}
    assert FICCO_FLAG_COUNTERS > F_RS + G * (G - 1)
    return low

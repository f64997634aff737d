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

import os
from collections import Counter
from dataclasses import dataclass, field

from .domain import Collective, Scenario
from .routing import (ExecutionPlan, GatherSpec, GemmSpec, PlanError, ScatterSpec, ScheduleKind, TransferSpec,
                      build_plan)
from .runtime import (BUF_A, BUF_B, BUF_C, BUF_MC, BUF_MCV, BUF_NONE, BUF_WS, EPI_REDUCE, EPI_STORE, EPI_STORE_REMOTE,
                      EPI_STORE_SIGNAL, FICCO_HINT_A_EVICT_LAST,
                      FICCO_HINT_CORE_COPIES,
                      FICCO_WS_DATA_OFFSET, MAX_RECV, OP_BARRIER, OP_COPY, OP_NOTIFY, OP_RECORD,
                      OP_REDUCE_MC, OP_SIGNAL, OP_STREAM_WAIT, OP_WAIT, OP_WAIT_COUNTER, TILE_K, TILE_M,
                      TILE_WIDTHS, CopyOp,
                      Operand, PlanDesc, Tile)

# Flag words, relative to the run's parity block (one-shot words, include/ficco.h).
# [0, 256): cross-rank words, written by peers and reset by their consumer
F_PUB = 0        # 8-byte barrier words (byte r = rank r published this run's shard)   [0, 4)
F_DONE = 4       # 8-byte barrier words (byte r = rank r started this run; RS receive) [4, 8)
F_RINGN = 64     # + step i: the left neighbour holds the shard we pull at ring step i+1
# [256, 4096): run-local flags, reset when the run starts
F_LOCAL = 256    # the local shard sits in its own slot
F_XFER = 320     # + c*G + p: chunk c of rank p landed (p = own rank is set with LOCAL)
F_RING = 704     # + step i: ring step i landed
F_RS = 1024      # + chunk*(G-1) + slot: a peer's partial chunk landed (RS; with comm_agent='core' a tile count)
F_GO = 258       # RS core: the DONE barrier passed, owners' receive slots may be written (run-local)
EV_START = 0     # event slot: the cross-rank barrier passed
EV_RING = 1      # + (step-1)*split + part: shard-ring step fork / part-landed events (ring_split > 1)


def ring_split() -> int:
    """Copy-engine chains per shard-ring step (FICCO_RING_SPLIT, default 1): the step's shard
    is pulled as that many row blocks on parallel copy streams, joined before RING[i]."""
    return max(1, min(8, int(os.environ.get("FICCO_RING_SPLIT", "1"))))
MAX_WORLD = 16

ELT = 2  # bf16
A_PIN_BYTES = 32 << 20  # A operands up to this size are kept in L2 (evict_last) when re-read per column tile


def _agent_hint(comm_agent) -> int:
    """comm_agent (the reference's CommAgent, machines.py:48): 'dma' = copy engines, 'core' = SM copies."""
    agent = getattr(comm_agent, "value", comm_agent)
    if agent not in ("dma", "core"):
        raise ValueError(f"comm_agent must be 'dma' or 'core', got {comm_agent!r}")
    return FICCO_HINT_CORE_COPIES if agent == "core" else 0


@dataclass
class Lowered:
    """A rank's program, ready for ``runtime.Plan``."""

    ops: list[CopyOp] = field(default_factory=list)
    tiles: list[Tile] = field(default_factory=list)
    desc: PlanDesc = field(default_factory=PlanDesc)
    ws_bytes: int = FICCO_WS_DATA_OFFSET
    gather_off: int = 0      # byte offset of parity-0 gathered buffer in the workspace
    gather_par: int = 0      # parity stride
    send_off: int = 0        # all-to-all: parity-0 send area (G blocks, block d addressed to rank d)
    send_par: int = 0
    recv_off: int = 0
    recv_par: int = 0
    recv_slot: int = 0
    mc_bytes: int = 0        # comm_agent = nvls: bytes of the multicast-bound partial buffer
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


def _tile(a_row, b_row, c_row, c_col, rows, cols, flag=-1, fmask=0, kseg=0, kstride=0, mode=EPI_STORE, chunk=0,
          recv_row=0, a_src=0, b_src=0) -> Tile:
    t = Tile()
    t.a_row, t.b_row, t.c_row, t.c_col, t.recv_row = a_row, b_row, c_row, c_col, recv_row
    t.rows, t.cols, t.flag, t.fmask = rows, cols, flag, (fmask if flag >= 0 else 0)
    t.kseg, t.kstride, t.mode, t.chunk, t.a_src, t.b_src = kseg, kstride, mode, chunk, a_src, b_src
    return t


B200_SMS = 148
DEFAULT_CTA_GROUP = 2


def pair_tiles(tiles: list[Tile]) -> list[Tile]:
    """Re-order a 128-row tile list into CTA pairs (cta_group::2).

    Tiles (2p, 2p+1) of the result share b_row / c_col / cols (one 256 x TN
    UMMA over two independent 128-row A pieces); a tile is emitted with the next
    tile of the same column range, so the order stays close to plan order.
    Unmatched tiles get a padding partner (rows = 0: loads, no stores/signals)
    that inherits the partner's readiness gates: each CTA of a pair loads half
    of the B rows, so B-side gates (CP: the gathered K rows) bind both CTAs.
    """
    pending: dict[tuple, Tile] = {}
    out: list[Tile] = []
    for t in tiles:
        # REDUCE tiles stream extra (partial x identity) k-blocks: both CTAs must do them
        key = (t.b_row, t.c_col, t.cols, t.b_src, t.mode == EPI_REDUCE)
        mate = pending.pop(key, None)
        if mate is None:
            pending[key] = t
        else:
            out += [mate, t]
    for t in pending.values():
        # the padding CTA still loads half of B, so it must honour the same gates
        pad = _tile(t.a_row, t.b_row, t.c_row, t.c_col, 0, t.cols, t.flag, t.fmask, t.kseg, t.kstride,
                    a_src=t.a_src, b_src=t.b_src)
        if t.mode == EPI_REDUCE:  # same k-block stream (and receive-slot gates) as its partner
            pad.mode, pad.chunk, pad.recv_row = EPI_REDUCE, t.chunk, t.recv_row
        out += [t, pad]
    return out


def choose_tile_n(tiles_for_width, sms: int = B200_SMS) -> int:
    """Tile width (UMMA N, B box rows) minimising persistent-kernel waves x wave time.

    ``tiles_for_width(w)`` is the tile count at width w. A wave of the
    persistent kernel is ``sms`` tiles. A wave does NOT get proportionally
    shorter with narrower tiles: every tile streams its full 256 x K slab of A
    through L2 -> SMEM whatever its width, so a tile costs about w + 512
    (measured, interleaved: 8192^3 takes 720 / 795 / 904 / 1059 / 1266 us at
    w = 256 / 224 / 192 / 160 / 128; profiles/r02_experiments/tile_width_ab.json).
    E.g. C2's N = 3584 at 256 gives 896 tiles = 6.05 waves (7 issued), at 224
    1024 tiles = 6.92 -> 224; 4096^3 at 256 is 3.5 waves -> 256 (not 128).
    """
    best, best_w = None, TILE_WIDTHS[0]
    for w in TILE_WIDTHS:
        n = tiles_for_width(w)
        cost = -(-n // sms) * (w + 512)
        if best is None or cost < best - 1e-9:
            best, best_w = cost, w
    return best_w


W_ROW_MAJOR_BYTES = 32 << 20  # a weight up to this size stays L2-resident under a row-major raster
W_L2_BYTES = 64 << 20         # about half the L2: a weight this large never stays resident beside the streams
A_GROUP_BYTES = 32 << 20      # otherwise rows are rastered in groups whose A slice stays in L2


def raster(frags: list[tuple[int, int]], N: int, K: int, tn: int) -> list[tuple[int, int, int]]:
    """Tiles (m0, n0, rows) covering the row fragments ``frags`` x [0, N).

    Row-major while W [N, K] stays L2-resident beside the streams (up to 32 MiB: C2; each W tile
    then comes from L2 for every row block). A larger W is re-read from HBM by every wave (C3's
    59 MiB: 0.86 GB of DRAM reads; EP g14's 235 MB: 102 GB), so the 128-row blocks go in groups of
    A_GROUP_BYTES and each group sweeps N column-major: W is read once per group, the group's A rows
    stay in L2 (pinned evict_last; W evict_last too; the plain GEMM uses the same raster,
    ficco.cu raster_rows).
    """
    blocks = [(m0, min(TILE_M, s + c - m0)) for s, c in frags for m0 in range(s, s + c, TILE_M)]
    if N * K * ELT <= W_ROW_MAJOR_BYTES:
        return [(m0, n0, rows) for m0, rows in blocks for n0 in range(0, N, tn)]
    per = max(2, (A_GROUP_BYTES // (K * ELT)) // TILE_M // 2 * 2)  # whole CTA pairs per group
    # balance the groups over this run's blocks: a fragment of 1.25 groups as one group (its A slice a
    # little over budget) rather than a full group plus a sliver that streams all of W again
    ngroups = max(1, round(len(blocks) / per))
    per = -(-len(blocks) // ngroups)
    per += per % 2
    out = []
    for i in range(0, len(blocks), per):
        out += [(m0, n0, rows) for n0 in range(0, N, tn) for m0, rows in blocks[i:i + per]]
    return out


def _check_shape(m: int, n: int, k: int) -> None:
    if k % 8:
        raise PlanError(f"K={k} must be a multiple of 8 (16-byte TMA rows)")
    if n % 32:
        raise PlanError(f"N={n} must be a multiple of 32 (epilogue column granularity)")


def _my_gemms(plan: ExecutionPlan, rank: int) -> list[GemmSpec]:
    return [t.kind for t in plan.tasks if t.gpu == rank and isinstance(t.kind, GemmSpec)]


def _publish(ops: list, g: int, world: int, row_bytes: int, shard_rows: int, gather_off: int, par: int,
             src_buf: int, inplace: bool = False) -> None:
    """Local shard -> own slot of the gathered buffer (stream 0), then the publish barrier.

    The tile kernel reads the local rows in place from the call argument (the
    alternate operand map), so nothing local gates a tile: the copy exists for
    the peers' pulls and for the gathered output. Stream 0 then runs the
    cross-rank barrier (each rank sets its byte in everyone's PUB word and waits
    for all bytes) and records EV_START, which every pull chain waits on.
    """
    if not inplace:  # in-place inputs already sit in the slot (see FiccoGroup.input_slot)
        ops.append(_op(OP_COPY, src_buf=src_buf, dst_buf=BUF_WS, src_off=0,
                       dst_off=gather_off + g * shard_rows * row_bytes, dst_par=par,
                       width=shard_rows * row_bytes, stream=0))
    ops.append(_op(OP_BARRIER, flag=F_PUB, stream=0))
    ops.append(_op(OP_RECORD, value=EV_START, stream=0))


def slab_split(G: int) -> int:
    """Copy-engine chains per uniform_fused_2d slab (FICCO_2D_SPLIT, default 1): each R x b slab pull is
    cut into that many row blocks on parallel copy streams, joined before the slab's XFER flag
    (strided 2D copies run at about half the 1D rate on one engine)."""
    want = int(os.environ.get("FICCO_2D_SPLIT", "1"))
    return max(1, min(want, (MAX_WORLD - 2) // max(1, G - 1)))


EV_SLAB = 40     # + peer chain * (split - 1) + part - 1: uniform_fused_2d slab-part landed (slab_split > 1)


def coalesce_groups(G: int) -> list[list[int]]:
    """Rounds whose chunks of one peer are pulled by ONE copy (FICCO_COALESCE=1): {0}, {1}, {2, 3},
    {4..7}, ... The plan's routing and every tile's gate are unchanged (each round's flag is still set,
    right behind the copy that carries it); only consecutive chunks of the same peer, adjacent in memory,
    share a copy-engine copy. Early rounds stay single so the first remote tiles start as soon as
    possible; later ones land long before the GEMM reaches them (profiles/r02_experiments/)."""
    if os.environ.get("FICCO_COALESCE", "0") != "1":
        return [[c] for c in range(G)]
    groups, c, size = [], 0, 1
    while c < G:
        n = min(size, G - c)
        groups.append(list(range(c, c + n)))
        c += n
        if len(groups) >= 2:
            size *= 2
    return groups


def fine_chains() -> int:
    """Copy-engine chains of the fine-grain AG copy programs (FICCO_FINE_CHAINS, default 0 = one per peer)."""
    return max(0, min(15, int(os.environ.get("FICCO_FINE_CHAINS", "0"))))


def _peer_stream(p: int, g: int, chains: int = 0) -> int:
    """Copy stream pulling from (or pushing to) peer p: one copy-engine chain per peer (or `chains` shared)."""
    idx = p if p < g else p - 1
    return 1 + (idx % chains if chains else idx)


def lower_ag(plan: ExecutionPlan, rank: int, gathered: str = "A", alpha: float = 1.0, grid: int = 0,
             other_rows: int | None = None, cta_group: int = DEFAULT_CTA_GROUP, inplace: bool = False,
             comm_agent: str = "dma") -> Lowered:
    """All-gather -> GEMM family (AG->GEMM and the CP KV-gather -> QK^T).

    gathered="A": C[M,N] = A_all[M,K] @ W[N,K]^T; call args (a=A_shard[R,K], b=W, c=C).
    gathered="B": S[Q,M] = alpha * Q[Q,K] @ K_all[M,K]^T; call args (a=Q, b=K_shard[R,K], c=S);
                  the plan's M rows (kv tokens) become output columns; ``other_rows`` = Q.

    A scenario whose collective is ``all_to_all`` (EP dispatch -> expert GEMM; the
    reference plans it exactly like all-gather, core.py:31-33) lowers
    the same routing with per-destination sources: the call argument a is this
    rank's send buffer [M, K] = G blocks of R rows, block d addressed to rank d;
    rank g's gathered rows p*R.. are peer p's block g. The ring schedule pulls each
    step's block straight from its origin (a block is addressed to one rank, so the
    plan's store-and-forward through the left neighbour becomes a direct NVSwitch
    pull with the same step order).
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
    a2a = sc.collective is Collective.ALL_TO_ALL
    if a2a and (gathered != "A" or inplace):
        raise PlanError("all_to_all lowers the gathered-A form from a call-argument send buffer")
    low = Lowered()
    low.gather_off = FICCO_WS_DATA_OFFSET
    low.gather_par = M * row_bytes
    low.ws_bytes = FICCO_WS_DATA_OFFSET + 2 * low.gather_par
    if a2a:  # send area (both parities): the peers pull their blocks from it
        low.send_off, low.send_par = low.ws_bytes, M * row_bytes
        low.ws_bytes += 2 * low.send_par
    ops = low.ops
    src_buf = BUF_A if gathered == "A" else BUF_B
    if G > MAX_WORLD:
        raise PlanError(f"at most {MAX_WORLD} ranks")
    if a2a:
        ops.append(_op(OP_COPY, src_buf=BUF_A, dst_buf=BUF_WS, dst_off=low.send_off, dst_par=low.send_par,
                       width=M * row_bytes, stream=0))
        ops.append(_op(OP_BARRIER, flag=F_PUB, stream=0))
        ops.append(_op(OP_RECORD, value=EV_START, stream=0))
        # own block -> own slot of the gathered (dispatched) buffer; tiles read it in place
        ops.append(_op(OP_COPY, src_buf=BUF_A, dst_buf=BUF_WS, src_off=g * R * row_bytes,
                       dst_off=low.gather_off + g * R * row_bytes, dst_par=low.gather_par, width=R * row_bytes,
                       stream=0))
    else:
        _publish(ops, g, G, row_bytes, R, low.gather_off, low.gather_par, src_buf, inplace)

    def pull(p: int, row0: int, nrows: int, stream: int) -> CopyOp:
        off = low.gather_off + row0 * row_bytes
        if a2a:  # peer p's block for this rank, same row offset inside the block
            src = low.send_off + (g * R + row0 - p * R) * row_bytes
            return _op(OP_COPY, peer=p, src_buf=BUF_WS, dst_buf=BUF_WS, src_off=src, dst_off=off,
                       src_par=low.send_par, dst_par=low.gather_par, width=nrows * row_bytes, stream=stream)
        return _op(OP_COPY, peer=p, src_buf=BUF_WS, dst_buf=BUF_WS, src_off=off, dst_off=off,
                   src_par=low.gather_par, dst_par=low.gather_par, width=nrows * row_bytes, stream=stream)

    # ---- copy program: the plan's TransferSpecs arriving at this rank, one pull chain per source peer
    xfers = [t.kind for t in plan.tasks if isinstance(t.kind, TransferSpec) and t.kind.dst == g]
    kseg = 0
    if kind is ScheduleKind.SHARD_OVERLAP_P2P and a2a:
        # ring step order, each step's block pulled directly from its origin rank (g - i)
        ops.append(_op(OP_STREAM_WAIT, value=EV_START, stream=1))
        for x in xfers:
            i = x.round_idx + 1
            src = (g - i) % G
            ops.append(pull(src, src * R, R, 1))
            ops.append(_op(OP_SIGNAL, flag=F_RING + i, stream=1))
    elif kind is ScheduleKind.SHARD_OVERLAP_P2P:
        # store-and-forward ring on one chain: step i pulls shard (g-i) from the left neighbour
        right = (g + 1) % G
        ops.append(_op(OP_STREAM_WAIT, value=EV_START, stream=1))
        ops.append(_op(OP_NOTIFY, peer=right, flag=F_RINGN + 0, stream=1))
        split = ring_split()
        bounds = [R * j // split for j in range(split + 1)]
        for x in xfers:
            i = x.round_idx + 1
            shard = (g - i) % G
            ops.append(_op(OP_WAIT, flag=F_RINGN + i - 1, stream=1))
            if split == 1:
                ops.append(pull(x.src, shard * R, R, 1))
            else:  # the shard as `split` row blocks on parallel copy streams 1, 2, ..., joined on stream 1
                ev = EV_RING + (i - 1) * split
                ops.append(_op(OP_RECORD, value=ev, stream=1))
                for j in range(split):
                    st = 1 + j
                    if j:
                        ops.append(_op(OP_STREAM_WAIT, value=ev, stream=st))
                    ops.append(pull(x.src, shard * R + bounds[j], bounds[j + 1] - bounds[j], st))
                    if j:
                        ops.append(_op(OP_RECORD, value=ev + j, stream=st))
                for j in range(1, split):
                    ops.append(_op(OP_STREAM_WAIT, value=ev + j, stream=1))
            ops.append(_op(OP_SIGNAL, flag=F_RING + i, stream=1))
            if i < G - 1:
                ops.append(_op(OP_NOTIFY, peer=right, flag=F_RINGN + i, stream=1))
    else:
        started: set[int] = set()
        if kind is ScheduleKind.UNIFORM_FUSED_2D:
            b = K // G
            if b % TILE_K:
                raise PlanError(f"uniform_fused_2d on B200 needs K/G={b} to be a multiple of {TILE_K}")
            kseg = b // TILE_K
        chains = fine_chains()
        group_of = {c: grp for grp in coalesce_groups(G) for c in grp}
        if kind is ScheduleKind.SERIAL or slab_split(G) > 1:
            group_of = {c: [c] for c in range(G)}
        for x in xfers:
            st = _peer_stream(x.src, g, chains)
            if st not in started:
                ops.append(_op(OP_STREAM_WAIT, value=EV_START, stream=st))
                started.add(st)
            c = x.round_idx
            rounds = group_of.get(c, [c])
            if kind is not ScheduleKind.SERIAL and len(rounds) > 1:
                if c != rounds[0]:
                    continue  # pulled with its group's first round
                n = len(rounds)
                if kind is ScheduleKind.UNIFORM_FUSED_2D:
                    b = K // G
                    off = low.gather_off + x.src * R * row_bytes + c * b * ELT
                    src, spar = (low.send_off + g * R * row_bytes + c * b * ELT, low.send_par) if a2a else \
                        (off, low.gather_par)
                    ops.append(_op(OP_COPY, peer=x.src, src_buf=BUF_WS, dst_buf=BUF_WS, src_off=src, dst_off=off,
                                   src_par=spar, dst_par=low.gather_par, width=n * b * ELT, height=R,
                                   src_pitch=row_bytes, dst_pitch=row_bytes, stream=st))
                else:
                    r = M // (G * G)
                    ops.append(pull(x.src, x.src * R + c * r, n * r, st))
                for cc in rounds:
                    ops.append(_op(OP_SIGNAL, flag=F_XFER + cc * G + x.src, stream=st))
                continue
            if kind is ScheduleKind.SERIAL:
                ops.append(pull(x.src, x.src * R, R, st))
            elif kind is ScheduleKind.UNIFORM_FUSED_2D:
                b = K // G
                off = low.gather_off + x.src * R * row_bytes + c * b * ELT
                src, spar = (low.send_off + g * R * row_bytes + c * b * ELT, low.send_par) if a2a else \
                    (off, low.gather_par)
                split = slab_split(G)
                bounds = [R * j // split for j in range(split + 1)]
                chain = st - 1
                for j in range(split - 1, -1, -1):  # helper parts first, the chain's own part last
                    sj = st + j * (G - 1)
                    if j and sj not in started:
                        ops.append(_op(OP_STREAM_WAIT, value=EV_START, stream=sj))
                        started.add(sj)
                    h = bounds[j + 1] - bounds[j]
                    ops.append(_op(OP_COPY, peer=x.src, src_buf=BUF_WS, dst_buf=BUF_WS,
                                   src_off=src + bounds[j] * row_bytes, dst_off=off + bounds[j] * row_bytes,
                                   src_par=spar, dst_par=low.gather_par, width=b * ELT, height=h,
                                   src_pitch=row_bytes, dst_pitch=row_bytes, stream=sj))
                    if j:
                        ops.append(_op(OP_RECORD, value=EV_SLAB + chain * (split - 1) + j - 1, stream=sj))
                for j in range(1, split):
                    ops.append(_op(OP_STREAM_WAIT, value=EV_SLAB + chain * (split - 1) + j - 1, stream=st))
            else:
                r = M // (G * G)
                ops.append(pull(x.src, x.src * R + c * r, r, st))
            ops.append(_op(OP_SIGNAL, flag=F_XFER + c * G + x.src, stream=st))

    # ---- tile program: this rank's GemmSpecs in plan order, each fragment gated by the flags it reads
    r_chunk = M // (G * G)

    peers_mask = ((1 << G) - 1) & ~(1 << g)

    def gate(start: int) -> tuple[int, int, int, int]:
        """(flag, fmask, kseg, kstride) for rows starting at `start` (one owner)."""
        owner = start // R
        if kind is ScheduleKind.UNIFORM_FUSED_1D:       # the step waits for its whole round (the gather)
            c = (start - owner * R) // r_chunk
            return F_XFER + c * G, peers_mask, 0, 0
        if owner == g:
            return -1, 0, 0, 0                           # local rows: read in place, no wait
        if kind is ScheduleKind.SERIAL:
            return F_XFER, peers_mask, 0, 0              # the whole all-gather
        if kind is ScheduleKind.SHARD_OVERLAP_P2P:
            return F_RING + (g - owner) % G, 1, 0, 0
        if kind is ScheduleKind.UNIFORM_FUSED_2D:
            return F_XFER + owner, 1, kseg, G            # k-segment c waits chunk (owner, c)
        c = (start - owner * R) // r_chunk
        if kind is ScheduleKind.HETERO_FUSED_1D:
            return F_XFER + c * G, peers_mask, 0, 0      # one fused GEMM per round
        return F_XFER + c * G + owner, 1, 0, 0           # unfused: exactly its own chunk

    Q = other_rows if gathered == "B" else None
    if gathered == "B" and Q is None:
        raise ValueError("gathered='B' needs other_rows (query rows)")
    frag_lists = []
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
        frag_lists.extend(frags)

    def cdiv(a: int, b: int) -> int:
        return -(-a // b)

    units = B200_SMS // cta_group
    if gathered == "A":
        tn = choose_tile_n(lambda w: cdiv(sum(cdiv(c, TILE_M) for _, c in frag_lists), cta_group) * cdiv(N, w),
                           units)
    else:
        tn = choose_tile_n(lambda w: sum(cdiv(c, w) for _, c in frag_lists) * cdiv(cdiv(Q, TILE_M), cta_group),
                           units)
    tiles = low.tiles
    if gathered == "A" and N * K * ELT > W_ROW_MAJOR_BYTES and os.environ.get("FICCO_AG_GROUP_GATES", "1") != "0":
        # a W beyond the row-major budget is streamed once per row group, so the groups span fragments
        # of DIFFERENT gates (each tile keeps its own block's gate): per-gate rasters would sweep all of W
        # once per fine chunk (hetero_unfused C3': 56 x 117 MB; EP g14: 41 GB per op). The groups follow
        # plan order, so a group waits at most for the chunks of its own rows.
        info = {}
        for start, count in frag_lists:
            for m0 in range(start, start + count, TILE_M):
                info[m0] = (gate(start), start // R == g)
        for m0, n0, rows in raster(frag_lists, N, K, tn):
            (flag, fmask, ks, kstride), local = info[m0]
            shift = g * R if local else 0  # own-shard rows come from the call argument (alternate map)
            tiles.append(_tile(m0 - shift, n0, m0, n0, rows, min(tn, N - n0), flag, fmask, ks, kstride,
                               a_src=int(local)))
    elif gathered == "A":
        # consecutive fragments behind the same gate (one fused step, the serial gather) are one
        # raster: a large W is then streamed once per row group, not once per fragment
        runs: list[tuple[tuple, list[tuple[int, int]]]] = []
        for start, count in frag_lists:
            key = (gate(start), start // R == g)
            if runs and runs[-1][0] == key:
                runs[-1][1].append((start, count))
            else:
                runs.append((key, [(start, count)]))
        for ((flag, fmask, ks, kstride), local), frags in runs:
            shift = g * R if local else 0  # own-shard rows come from the call argument (alternate map)
            for m0, n0, rows in raster(frags, N, K, tn):
                tiles.append(_tile(m0 - shift, n0, m0, n0, rows, min(tn, N - n0), flag, fmask, ks, kstride,
                                   a_src=int(local)))
    if gathered == "B":
        # kv column blocks ("units", one B tile each) in plan order, each gated by the flags of its rows
        units = []
        for fi, (start, count) in enumerate(frag_lists):
            if count % 32:
                raise PlanError(f"gathered-B fragments must be multiples of 32 rows, got {count}")
            gt = gate(start)
            local = start // R == g  # rows of the own shard come from the call argument (alternate map)
            for n0 in range(start, start + count, tn):
                units.append((n0, min(tn, start + count - n0), gt, local, g * R if local else 0, fi))
        step = TILE_M * cta_group
        slots = B200_SMS // cta_group

        def emit(unit, mb, pad=False):
            n0, cols, (flag, fmask, ks, kstride), local, shift, _ = unit
            for m0 in range(mb, min(Q, mb + step), TILE_M):
                tiles.append(_tile(m0, n0 - shift, m0, n0, 0 if pad else min(TILE_M, Q - m0), cols, flag, fmask,
                                   ks, kstride, b_src=int(local)))

        if len(units) >= slots:
            # B-stationary: the persistent kernel hands pair-tile i to CTA pair i mod 74, so listing a
            # wave of 74 units query-block by query-block gives every pair ONE kv block for all its query
            # blocks. With K = d <= 256 the tile kernel then keeps those B rows in smem (b_resident) and
            # streams only Q: half the L2->SM bytes of this store-bound op. A last partial wave is
            # padded with load-only tiles (rows = 0) so the pair mapping stays aligned.
            for w0 in range(0, len(units), slots):
                wave = units[w0:w0 + slots]
                for mb in range(0, Q, step):
                    for u in wave:
                        emit(u, mb)
                    for _ in range(slots - len(wave)):
                        emit(wave[0], mb, pad=True)
        else:
            # few units: query-row-major inside each fragment (concurrent tiles write long contiguous row
            # segments of the score matrix); 256-row steps keep CTA-pair partners (m0, m0 + 128) adjacent
            for fi in range(len(frag_lists)):
                fr = [u for u in units if u[5] == fi]
                for mb in range(0, Q, step):
                    for u in fr:
                        emit(u, mb)

    if cta_group == 2:
        low.tiles[:] = pair_tiles(low.tiles)
    d = low.desc
    gat = _operand(BUF_WS, M, K, low.gather_off, low.gather_par)
    # local rows: read in place from the call argument, or from the own slot for in-place inputs
    own = _operand(BUF_WS, R, K, low.gather_off + g * R * row_bytes, low.gather_par) if inplace else None
    if gathered == "A":
        d.a, d.b, d.c = gat, _operand(BUF_B, N, K), _operand(BUF_C, M, N)
        # local rows: the own shard (all-gather) or the own block g of the send buffer (all-to-all)
        local_a = _operand(BUF_A, R, K, g * R * row_bytes if a2a else 0)
        d.a2, d.b2 = own or local_a, _operand(BUF_NONE, 0, 0)
    else:
        d.a, d.b, d.c = _operand(BUF_A, Q, K), gat, _operand(BUF_C, Q, M)
        d.a2, d.b2 = _operand(BUF_NONE, 0, 0), own or _operand(BUF_B, R, K)
    d.part = _operand(BUF_NONE, 0, 0)
    d.recv = _operand(BUF_NONE, 0, 0)
    d.k, d.alpha, d.grid, d.tile_n, d.cta_group = K, alpha, grid, tn, cta_group
    # a small A (CP: Q, a few MiB) is re-read by every column tile while the output streams
    # through L2 (4 GiB of scores in C4) — pin it (evict_last) instead of the default evict_first
    a_bytes = (Q if gathered == "B" else M) * K * ELT
    grouped = gathered == "A" and N * K * ELT > W_ROW_MAJOR_BYTES  # column-major raster (see raster)
    if os.environ.get("FICCO_A_EVICT_LAST", "auto") == "1" or (
            os.environ.get("FICCO_A_EVICT_LAST", "auto") == "auto" and (a_bytes <= A_PIN_BYTES or grouped)):
        d.hints |= FICCO_HINT_A_EVICT_LAST
    # W stays evict_last even when it exceeds L2: the group's row blocks re-read each column tile
    # (evict_first measured 2.3-4.6 % slower on C3 G2/G4, C3' and EP: r02_experiments/w_policy_ab.json)
    d.hints |= _agent_hint(comm_agent)
    low.notes = {"kind": kind.value, "rank": g, "world": G, "gathered": gathered, "inplace": inplace,
                 "comm_agent": comm_agent, "collective": sc.collective.value}
    return low


RS_KINDS = (ScheduleKind.SERIAL, ScheduleKind.SHARD_OVERLAP_P2P, ScheduleKind.UNIFORM_FUSED_1D,
            ScheduleKind.HETERO_FUSED_1D, ScheduleKind.HETERO_UNFUSED_1D, ScheduleKind.UNIFORM_FUSED_2D)


@dataclass(frozen=True)
class RSPiece:
    """One pushed block of a GEMM -> RS schedule: rows [row0, +nrows) x cols [col0, +ncols) of the
    partial P_g, owned by rank ``owner``; ``idx`` selects its landing words F_RS + idx*(G-1) + slot."""

    owner: int
    row0: int
    nrows: int
    col0: int
    ncols: int
    idx: int


def rs_pieces(scenario: Scenario, kind: ScheduleKind, rank: int):
    """The adjoint routing of ``kind`` for rank ``rank``: (emission order, push units).

    order: [(remote?, piece)] in tile order; units: [[pieces pushed together]] (dma agent).
    Time-reversal of the AG schedules (planner.py:170-390): where the AG schedule receives chunk
    (p, c) before the GEMM that reads it, the RS schedule computes the partial of chunk (q, c)
    before pushing it to its owner q, and the owner's own-rows tiles reduce last:

    serial            all remote shards, ONE push unit after the whole GEMM (planner.py:170-191)
    shard_overlap     shard ring reversed: step i computes owner (g+i)'s shard and pushes it
                      (whole shard, one unit per step), own shard last (planner.py:194-240)
    uniform_fused_1d  round c: chunk c of every remote owner (one unit), then the own chunk c
    hetero_fused_1d   all remote rounds (one unit per round), own shard last (planner.py:291-331)
    hetero_unfused_1d as fused, one unit per chunk (planner.py:332-347)
    uniform_fused_2d  the N-block adjoint of the K-block schedule (planner.py:351-390): round c
                      computes output column block c of every remote owner's rows (an R x N/G
                      slab, one unit), then the own slab c, which reduces as soon as round c landed
    """
    if kind not in RS_KINDS:
        raise PlanError(f"GEMM->reduce-scatter has no executable adjoint of {kind.value}")
    g, G = rank, scenario.n_gpus
    M, N = scenario.gemm.m, scenario.gemm.n
    if kind is ScheduleKind.UNIFORM_FUSED_2D:
        if M % G or N % G:
            raise PlanError(f"uniform_fused_2d (N-block) GEMM->RS needs M={M} and N={N} divisible by G={G}")
        if (N // G) % 32:
            raise PlanError(f"uniform_fused_2d (N-block) GEMM->RS needs N/G={N // G} to be a multiple of 32")
    elif kind in (ScheduleKind.SERIAL, ScheduleKind.SHARD_OVERLAP_P2P):
        build_plan(scenario, kind)  # M % G, exactly as the AG schedule
    else:
        build_plan(scenario, kind)  # M % G^2
    R = M // G
    remote = [(g + j) % G for j in range(1, G)]
    order: list[tuple[bool, RSPiece]] = []
    units: list[list[RSPiece]] = []
    if kind in (ScheduleKind.SERIAL, ScheduleKind.SHARD_OVERLAP_P2P):
        pcs = [RSPiece(q, q * R, R, 0, N, 0) for q in remote]
        order = [(True, pc) for pc in pcs] + [(False, RSPiece(g, g * R, R, 0, N, 0))]
        units = [pcs] if kind is ScheduleKind.SERIAL else [[pc] for pc in pcs]
        return order, units
    if kind is ScheduleKind.UNIFORM_FUSED_2D:
        b = N // G
        for c in range(G):
            pcs = [RSPiece(q, q * R, R, c * b, b, c) for q in remote]
            units.append(pcs)
            order += [(True, pc) for pc in pcs] + [(False, RSPiece(g, g * R, R, c * b, b, c))]
        return order, units
    r = M // (G * G)
    for c in range(G):
        pcs = [RSPiece(q, q * R + c * r, r, 0, N, c) for q in remote]
        units += [[pc] for pc in pcs] if kind is ScheduleKind.HETERO_UNFUSED_1D else [pcs]
        order += [(True, pc) for pc in pcs]
        if kind is ScheduleKind.UNIFORM_FUSED_1D:
            order.append((False, RSPiece(g, g * R + c * r, r, 0, N, c)))
    if kind is not ScheduleKind.UNIFORM_FUSED_1D:
        order += [(False, RSPiece(g, g * R + c * r, r, 0, N, c)) for c in range(G)]
    return order, units


def lower_rs(scenario: Scenario, kind: ScheduleKind, rank: int, grid: int = 0, virtual: bool = False,
             cta_group: int = DEFAULT_CTA_GROUP, comm_agent: str = "dma") -> Lowered:
    """GEMM -> reduce-scatter (not in the reference, parity unpinned).

    Rank g holds A_g [M, Kg] and W_g [N, Kg]; P_g = A_g @ W_g^T [M, N]; rank q
    ends with C_q = sum_g P_g[q*R:(q+1)*R] [R, N]. The schedule's pieces (``rs_pieces``):
    remote pieces' tiles store their partial and are counted; the copy stream pushes each
    finished unit into the owners' receive slots (copy engine) and notifies them; the
    owner's own-rows tiles (REDUCE) fold the G-1 received partials into the fp32
    accumulator (rank-ascending, one bf16 rounding) once their landing words are set.

    comm_agent='core' (the SM-driven variant, reference CommAgent.CORE): no
    partial buffer and no push copies. A remote piece's tile epilogue TMA-stores
    the partial straight into the owner's receive slot (peer memory over
    NVLink) and bumps the owner's per-(piece, sender) word; the owner reduces
    once that word reaches the sender's tile count (``rs_target``). Stores wait
    for the DONE barrier (flag F_GO), as the copy-engine pushes do.
    """
    if getattr(comm_agent, "value", comm_agent) == "nvls":
        return lower_rs_nvls(scenario, kind, rank, grid=grid, virtual=virtual, cta_group=cta_group)
    order, units = rs_pieces(scenario, kind, rank)
    g, G = rank, scenario.n_gpus
    M, N, K = scenario.gemm.m, scenario.gemm.n, scenario.gemm.k
    _check_shape(M, N, K)
    if G - 1 > MAX_RECV or G > MAX_WORLD:
        raise PlanError(f"at most {MAX_RECV + 1} ranks")
    R = M // G
    row_bytes = N * ELT
    low = Lowered()
    direct = getattr(comm_agent, "value", comm_agent) == "core"
    part_off = FICCO_WS_DATA_OFFSET
    low.recv_off = part_off + (0 if direct else M * row_bytes)  # direct stores need no partial buffer
    low.recv_slot = R * row_bytes
    low.recv_par = 0  # single buffer: a peer pushes run e only after our DONE(e), i.e. after run e-1 finished
    low.ws_bytes = low.recv_off + (G - 1) * low.recv_slot
    ops, tiles = low.ops, low.tiles
    _agent_hint(comm_agent)  # validates the name

    def slot_of(src: int, owner: int) -> int:
        return src if src < owner else src - 1

    def cdiv(a: int, b: int) -> int:
        return -(-a // b)

    shape0 = order[0][1]
    tn = choose_tile_n(lambda w: cdiv(len(order) * cdiv(shape0.nrows, TILE_M), cta_group) * cdiv(shape0.ncols, w),
                       B200_SMS // cta_group)
    tiles_per_piece = cdiv(shape0.nrows, TILE_M) * cdiv(shape0.ncols, tn)
    unit_of = {pc: uid for uid, pcs in enumerate(units) for pc in pcs}

    # Tile order: the schedule's pieces in order. While W stays L2-resident (<= 32 MiB) each piece is
    # row-major. A larger W would be re-read from HBM by every wave (C3 at G = 8: 59 MB; at G = 2: 235 MB),
    # so each run of full-width pieces of the same role (remote / own) is cut into 128-row blocks, the
    # blocks go in balanced groups of <= A_GROUP_BYTES of A, and each group sweeps N column-major with
    # its A rows pinned in L2 (as lowering.raster does for the AG side and ficco.cu raster_rows for the
    # plain GEMM).
    grouped_rs = N * K * ELT > W_ROW_MAJOR_BYTES and os.environ.get("FICCO_RS_GROUP", "1") != "0"
    budget = max(2, A_GROUP_BYTES // (K * ELT) // TILE_M // 2 * 2)  # 128-row blocks per group (even)
    seq: list[tuple[bool, RSPiece, int, int, int, int]] = []  # (remote, piece, m0, rows, n0, cols)
    i = 0
    while i < len(order):
        j = i + 1
        full = order[i][1].ncols == N
        while grouped_rs and full and j < len(order) and order[j][0] == order[i][0] and order[j][1].ncols == N:
            j += 1
        run = [pc for _, pc in order[i:j]]
        blocks = [(pc, m0, min(TILE_M, pc.row0 + pc.nrows - m0)) for pc in run
                  for m0 in range(pc.row0, pc.row0 + pc.nrows, TILE_M)]
        if not (grouped_rs and full) or len(blocks) <= 2:
            seq += [(order[i][0], pc, m0, rows, n0, min(tn, pc.col0 + pc.ncols - n0)) for pc, m0, rows in blocks
                    for n0 in range(pc.col0, pc.col0 + pc.ncols, tn)]
        else:
            per = -(-len(blocks) // -(-len(blocks) // budget))
            per += per % 2
            for x in range(0, len(blocks), per):
                seq += [(order[i][0], pc, m0, rows, n0, min(tn, N - n0)) for n0 in range(0, N, tn)
                        for pc, m0, rows in blocks[x:x + per]]
        i = j

    for is_remote, pc, m0, rows, n0, cols in seq:
        if is_remote and direct:
            tiles.append(_tile(m0, n0, m0 - pc.owner * R, n0, rows, cols, mode=EPI_STORE_REMOTE,
                               chunk=pc.owner, recv_row=F_RS + pc.idx * (G - 1) + slot_of(g, pc.owner)))
        elif is_remote:
            tiles.append(_tile(m0, n0, m0, n0, rows, cols, mode=EPI_STORE_SIGNAL, chunk=unit_of[pc]))
        else:
            local = m0 - g * R
            tiles.append(_tile(m0, n0, local, n0, rows, cols, mode=EPI_REDUCE, chunk=pc.idx,
                               recv_row=local))

    if cta_group == 2:
        tiles[:] = pair_tiles(tiles)

    # copy program. Stream 0: DONE barrier (every peer has started this run, so its
    # receive slots are free), then one counter wait per push unit, each published as
    # an event the owners' push chains (one per peer q) wait on before their copies.
    n_idx = 1 + max(pc.idx for _, pc in order)
    if virtual:  # stand-in peers never push: their partials are pre-loaded, mark them all landed at once
        ops.append(_op(OP_SIGNAL, flag=F_RS, value=n_idx * (G - 1), stream=0))
    ops.append(_op(OP_BARRIER, flag=F_DONE, stream=0))
    if direct:  # the tile epilogues push: release them, nothing else to copy
        ops.append(_op(OP_SIGNAL, flag=F_GO, stream=0))
        units = []
    else:
        ops.append(_op(OP_RECORD, value=EV_START, stream=0))
        for q in range(G):
            if q != g:
                ops.append(_op(OP_STREAM_WAIT, value=EV_START, stream=_peer_stream(q, g)))
    for uid, pcs in enumerate(units):
        slot = 1 + uid % 63
        ops.append(_op(OP_WAIT_COUNTER, flag=uid, value=tiles_per_piece * len(pcs), stream=0))
        ops.append(_op(OP_RECORD, value=slot, stream=0))
        for pc in pcs:
            q = pc.owner
            st = _peer_stream(q, g)
            ops.append(_op(OP_STREAM_WAIT, value=slot, stream=st))
            src = part_off + pc.row0 * row_bytes + pc.col0 * ELT
            dst = low.recv_off + slot_of(g, q) * low.recv_slot + (pc.row0 - q * R) * row_bytes + pc.col0 * ELT
            if pc.ncols == N:
                ops.append(_op(OP_COPY, src_buf=BUF_WS, dst_buf=BUF_WS, dst_peer=q, src_off=src, dst_off=dst,
                               width=pc.nrows * row_bytes, stream=st))
            else:  # an R x N/G column slab: one 2D copy-engine copy
                ops.append(_op(OP_COPY, src_buf=BUF_WS, dst_buf=BUF_WS, dst_peer=q, src_off=src, dst_off=dst,
                               width=pc.ncols * ELT, height=pc.nrows, src_pitch=row_bytes, dst_pitch=row_bytes,
                               stream=st))
            ops.append(_op(OP_NOTIFY, peer=q, flag=F_RS + pc.idx * (G - 1) + slot_of(g, q), stream=st))

    d = low.desc
    d.a, d.b = _operand(BUF_A, M, K), _operand(BUF_B, N, K)
    d.c = _operand(BUF_C, R, N)
    d.part = _operand(BUF_NONE, 0, 0) if direct else _operand(BUF_WS, M, N, part_off)
    if direct:
        per_word = Counter((t.chunk, t.recv_row) for t in tiles if t.mode == EPI_STORE_REMOTE)
        if len(set(per_word.values())) != 1:
            raise PlanError("uneven STORE_REMOTE tile counts per (piece, sender)")
        d.rs_target, d.go_flag = next(iter(per_word.values())), F_GO
    d.recv = _operand(BUF_WS, R, N, low.recv_off, low.recv_par)
    d.a2, d.b2 = _operand(BUF_NONE, 0, 0), _operand(BUF_NONE, 0, 0)
    d.recv_slot, d.n_recv, d.rs_flag0 = low.recv_slot, G - 1, F_RS
    d.n_counters = len(units)
    d.k, d.alpha, d.grid, d.tile_n, d.cta_group = K, 1.0, grid, tn, cta_group
    if grouped_rs and os.environ.get("FICCO_A_EVICT_LAST", "auto") != "0":
        d.hints |= FICCO_HINT_A_EVICT_LAST  # the group's A slice stays in L2 while it sweeps N

    if not direct:
        d.hints |= _agent_hint(comm_agent)
    if len(units) >= 4096 - 1:
        raise PlanError("too many push units")
    if F_RS + n_idx * (G - 1) >= 4096:
        raise PlanError("too many ranks for the RS flag area")
    low.notes = {"kind": kind.value, "rank": g, "world": G, "op": "rs", "units": len(units),
                 "tiles_per_chunk": tiles_per_piece, "comm_agent": comm_agent}
    return low


def lower_rs_nvls(scenario: Scenario, kind: ScheduleKind, rank: int, grid: int = 0, virtual: bool = False,
                  cta_group: int = DEFAULT_CTA_GROUP) -> Lowered:
    """GEMM -> reduce-scatter with comm_agent='nvls' (in-switch reduction).

    Every rank stores its WHOLE partial P_g [M, N] (bf16) into the memory it bound to the group's NVLS
    multicast object (FICCO_BUF_MC); nothing is copied. When a piece's tiles are stored (unit counter) the
    copy program notifies the piece's owner; once the owner has all G-1 notifications for its piece c and
    its own tiles of that piece are stored, a REDUCE_MC op reads the rows through the multicast VA
    (multimem.ld_reduce.add.acc::f32.bf16x2): the NVSwitch returns the sum over every rank's copy, fp32
    accumulation of the G bf16 partials (the owner's included), one bf16 rounding, written to C. The tile
    and notification order follow the schedule's adjoint routing (rs_pieces). Partial stores wait for the
    DONE barrier (go flag), so a rank never overwrites partials an owner is still reducing from the
    previous call. Needs real ranks on distinct GPUs with multicast access (no virtual peers).
    """
    if virtual:
        raise PlanError("comm_agent='nvls' needs real ranks on distinct GPUs (one multicast object over their "
                        "memory); virtual peers have none")
    order, units = rs_pieces(scenario, kind, rank)
    g, G = rank, scenario.n_gpus
    M, N, K = scenario.gemm.m, scenario.gemm.n, scenario.gemm.k
    _check_shape(M, N, K)
    if N % 8:
        raise PlanError("nvls reduce reads 16-byte vectors: N must be a multiple of 8")
    if G - 1 > MAX_RECV or G > MAX_WORLD:
        raise PlanError(f"at most {MAX_RECV + 1} ranks")
    R = M // G
    row_bytes = N * ELT
    low = Lowered()
    low.ws_bytes = FICCO_WS_DATA_OFFSET
    low.mc_bytes = M * row_bytes
    ops, tiles = low.ops, low.tiles

    def slot_of(src: int, owner: int) -> int:
        return src if src < owner else src - 1

    def cdiv(a: int, b: int) -> int:
        return -(-a // b)

    own = [pc for rem, pc in order if not rem]
    all_units = units + [[pc] for pc in own]  # own pieces are units too: their counter gates the reduce
    unit_of = {pc: uid for uid, pcs in enumerate(all_units) for pc in pcs}
    shape0 = order[0][1]
    tn = choose_tile_n(lambda w: cdiv(len(order) * cdiv(shape0.nrows, TILE_M), cta_group) * cdiv(shape0.ncols, w),
                       B200_SMS // cta_group)
    tiles_per_piece = cdiv(shape0.nrows, TILE_M) * cdiv(shape0.ncols, tn)
    for _, pc in order:
        for m0 in range(pc.row0, pc.row0 + pc.nrows, TILE_M):
            rows = min(TILE_M, pc.row0 + pc.nrows - m0)
            for n0 in range(pc.col0, pc.col0 + pc.ncols, tn):
                tiles.append(_tile(m0, n0, m0, n0, rows, min(tn, pc.col0 + pc.ncols - n0), mode=EPI_STORE_SIGNAL,
                                   chunk=unit_of[pc]))
    if cta_group == 2:
        tiles[:] = pair_tiles(tiles)

    # stream 0: DONE barrier -> release the partial stores (go) -> notify each owner as its units complete
    ops.append(_op(OP_BARRIER, flag=F_DONE, stream=0))
    ops.append(_op(OP_SIGNAL, flag=F_GO, stream=0))
    for uid, pcs in enumerate(units):
        ops.append(_op(OP_WAIT_COUNTER, flag=uid, value=tiles_per_piece * len(pcs), stream=0))
        for pc in pcs:
            ops.append(_op(OP_NOTIFY, peer=pc.owner, flag=F_RS + pc.idx * (G - 1) + slot_of(g, pc.owner), stream=0))
    # stream 1: per own piece, wait for it everywhere, then reduce it in the switch into C
    for pc in own:
        ops.append(_op(OP_WAIT_COUNTER, flag=unit_of[pc], value=tiles_per_piece, stream=1))
        for j in range(G - 1):
            ops.append(_op(OP_WAIT, flag=F_RS + pc.idx * (G - 1) + j, stream=1))
        ops.append(_op(OP_REDUCE_MC, src_buf=BUF_MCV, dst_buf=BUF_C, src_off=pc.row0 * row_bytes + pc.col0 * ELT,
                       dst_off=(pc.row0 - g * R) * row_bytes + pc.col0 * ELT, width=pc.ncols * ELT, height=pc.nrows,
                       src_pitch=row_bytes, dst_pitch=row_bytes, stream=1))

    d = low.desc
    d.a, d.b = _operand(BUF_A, M, K), _operand(BUF_B, N, K)
    d.c = _operand(BUF_C, R, N)
    d.part = _operand(BUF_MC, M, N, 0)
    d.recv = _operand(BUF_NONE, 0, 0)
    d.a2, d.b2 = _operand(BUF_NONE, 0, 0), _operand(BUF_NONE, 0, 0)
    d.n_counters = len(all_units)
    d.go_flag = F_GO
    d.k, d.alpha, d.grid, d.tile_n, d.cta_group = K, 1.0, grid, tn, cta_group
    if len(all_units) >= 4096 - 2048 or F_RS + G * (G - 1) >= 2048:
        raise PlanError("too many push units / ranks for the flag block")
    low.notes = {"kind": kind.value, "rank": g, "world": G, "op": "rs", "units": len(all_units),
                 "tiles_per_chunk": tiles_per_piece, "comm_agent": "nvls"}
    return low

"""Multi-rank interpreter of lowered FiCCO programs (test infrastructure, CPU only).

Executes G ranks' copy programs (include/ficco.h opcodes) and tile programs on
numpy byte buffers under a randomised scheduler, with the executor's
semantics:

* per rank, runs are sequential (run r+1 starts after every stream and the
  tile kernel of run r finished), ranks drift freely against each other;
* within a run, ops of one copy stream execute in order; streams, the tile
  kernel's tiles and other ranks interleave arbitrarily (random choice among
  everything runnable), so any ordering the hardware could produce between
  synchronisation points can be drawn;
* run r uses flag block / workspace parity r & 1; the other block's run-local
  words are cleared at some random point during run r (side-stream memset);
* COPY moves bytes at the instant it executes — reading a slot before its
  producer wrote it yields stale bytes, which the final comparison catches.

It validates the cross-rank protocol (publish / DONE barriers, ring
notifications, one-shot parity flags, counter-gated pushes, receive-buffer
reuse) that cannot be exercised with a single physical GPU, and the tile
programs' coverage and gating.
"""

from __future__ import annotations

import random

import numpy as np

from paper_2512_10236_b200.runtime import (BUF_A, BUF_B, BUF_C, BUF_MC, BUF_MCV, BUF_NONE, BUF_WS, EPI_REDUCE,
                                           EPI_STORE,
                                           EPI_STORE_REMOTE, EPI_STORE_SIGNAL, FICCO_FLAG_BLOCK, FICCO_FLAG_COUNTERS,
                                           FICCO_FLAG_RUN_LOCAL, OP_BARRIER, OP_COPY, OP_NOTIFY, OP_RECORD,
                                           OP_REDUCE_MC, OP_SIGNAL, OP_STREAM_WAIT, OP_WAIT, OP_WAIT_COUNTER,
                                           TILE_K)


class Deadlock(AssertionError):
    pass


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 (already bf16-representable) -> raw bf16 bits (uint16)."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def bits_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


class Rank:
    def __init__(self, g: int, ws_bytes: int, mc_bytes: int = 0):
        self.g = g
        self.ws = np.zeros(ws_bytes, dtype=np.uint8)
        self.mc = np.zeros(mc_bytes, dtype=np.uint8)  # memory bound to the NVLS multicast object
        self.flags = self.ws[: 16384 * 4].view(np.uint32)

    def block(self, parity: int) -> np.ndarray:
        return self.flags[parity * FICCO_FLAG_BLOCK:(parity + 1) * FICCO_FLAG_BLOCK]


class World:
    """G ranks executing `runs` consecutive calls of their lowered programs."""

    def __init__(self, lowered: list, args_per_run: list, seed: int = 0):
        self.low = lowered
        self.G = len(lowered)
        self.ranks = [Rank(g, lowered[g].ws_bytes, getattr(lowered[g], "mc_bytes", 0)) for g in range(self.G)]
        self.args = args_per_run  # args[run][rank] = dict(a=ndarray uint16 2D, b=..., c=...)
        self.rng = random.Random(seed)
        self.steps = 0

    # ---------------------------------------------------------------- buffers
    def _buf(self, rank: int, run: int, buf: int, peer: int) -> np.ndarray:
        if buf == BUF_WS:
            return self.ranks[rank if peer < 0 else peer].ws
        if buf == BUF_MC:
            return self.ranks[rank].mc
        key = {BUF_A: "a", BUF_B: "b", BUF_C: "c"}[buf]
        return self.args[run][rank][key].view(np.uint8).reshape(-1)

    def _copy(self, rank: int, run: int, op) -> None:
        par = run & 1
        src = self._buf(rank, run, op.src_buf, op.peer)
        dst = self._buf(rank, run, op.dst_buf, op.dst_peer)
        so = op.src_off + (op.src_par if par else 0)
        do = op.dst_off + (op.dst_par if par else 0)
        h = max(1, op.height)
        sp = op.src_pitch if h > 1 else op.width
        dp = op.dst_pitch if h > 1 else op.width
        for i in range(h):
            dst[do + i * dp: do + i * dp + op.width] = src[so + i * sp: so + i * sp + op.width]

    def _reduce_mc(self, rank: int, run: int, op) -> None:
        """NVSwitch in-switch reduction: every rank's multicast-bound copy of the rows, fp32 sum, one bf16
        rounding (multimem.ld_reduce.add.acc::f32.bf16x2)."""
        dst = self._buf(rank, run, op.dst_buf, op.dst_peer)
        h = max(1, op.height)
        for i in range(h):
            so = op.src_off + i * op.src_pitch
            acc = np.zeros(op.width // 2, dtype=np.float32)
            for rk in self.ranks:
                acc = acc + bits_f32(rk.mc[so:so + op.width].view(np.uint16))
            do = op.dst_off + i * op.dst_pitch
            dst[do:do + op.width] = bf16_bits(round_bf16(acc)).view(np.uint8)

    def _operand(self, rank: int, run: int, od) -> np.ndarray | None:
        if od.buf == BUF_NONE:
            return None
        base = self._buf(rank, run, od.buf, -1)
        off = od.off + (od.par if run & 1 else 0)
        return base[off: off + od.rows * od.ld * 2].view(np.uint16).reshape(od.rows, od.ld)

    # ---------------------------------------------------------------- tiles
    def _tile_ready(self, rank: int, run: int, t, kseg_done: int) -> bool:
        if t.flag < 0:
            return True
        blk = self.ranks[rank].block(run & 1)
        base = t.flag + (kseg_done * t.kstride if t.kseg else 0)
        return all(blk[base + i] != 0 for i in range(16) if t.fmask >> i & 1)

    def _run_tile(self, rank: int, run: int, t) -> None:
        d = self.low[rank].desc
        K = d.k
        A = self._operand(rank, run, d.a2 if t.a_src else d.a)
        B = self._operand(rank, run, d.b2 if t.b_src else d.b)
        if t.rows == 0:
            return
        a = bits_f32(A[t.a_row:t.a_row + t.rows, :K])
        b = bits_f32(B[t.b_row:t.b_row + t.cols, :K])
        acc = a @ b.T
        if t.mode == EPI_STORE:
            acc = acc * np.float32(d.alpha)
            out = self._operand(rank, run, d.c)
        elif t.mode == EPI_STORE_SIGNAL:
            out = self._operand(rank, run, d.part)
        elif t.mode == EPI_STORE_REMOTE:  # straight into owner t.chunk's receive slot for this rank
            q = t.chunk
            slot = rank if rank < q else rank - 1
            base = self.ranks[q].ws
            off = d.recv.off + (d.recv.par if run & 1 else 0) + slot * d.recv_slot
            out = base[off: off + d.recv.rows * d.recv.ld * 2].view(np.uint16).reshape(d.recv.rows, d.recv.ld)
        else:
            blk = self.ranks[rank].block(run & 1)
            for j in range(d.n_recv):
                assert blk[d.rs_flag0 + t.chunk * d.n_recv + j] >= max(1, d.rs_target), \
                    "REDUCE before its partials landed"
                base = self._buf(rank, run, d.recv.buf, -1)
                off = d.recv.off + (d.recv.par if run & 1 else 0) + j * d.recv_slot
                slot = base[off: off + d.recv.rows * d.recv.ld * 2].view(np.uint16).reshape(d.recv.rows, d.recv.ld)
                acc = acc + bits_f32(slot[t.recv_row:t.recv_row + t.rows, t.c_col:t.c_col + t.cols])
            out = self._operand(rank, run, d.c)
        out[t.c_row:t.c_row + t.rows, t.c_col:t.c_col + t.cols] = bf16_bits(round_bf16(acc))
        if t.mode == EPI_STORE_SIGNAL:
            blk = self.ranks[rank].block(run & 1)
            blk[FICCO_FLAG_COUNTERS + t.chunk] += 1
        elif t.mode == EPI_STORE_REMOTE:
            self.ranks[t.chunk].block(run & 1)[t.recv_row] += 1

    # ---------------------------------------------------------------- driver
    def run(self, runs: int) -> None:
        G = self.G
        state = []  # per rank: current run, stream positions, tile states
        for g in range(G):
            state.append({"run": -1})
        for g in range(G):
            self._start(g, state[g])
        while any(st["run"] < runs for st in state):
            actions = []
            for g in range(G):
                st = state[g]
                if st["run"] >= runs:
                    continue
                actions += self._runnable(g, st)
            if not actions:
                raise Deadlock(f"no runnable action; runs={[s['run'] for s in state]}")
            act = self.rng.choice(actions)
            act()
            self.steps += 1
            for g in range(G):
                st = state[g]
                if st["run"] < runs and self._finished(st):
                    self.on_run_done(g, st["run"])
                    self._start(g, state[g])

    def on_run_done(self, rank: int, run: int) -> None:  # hook for checks
        pass

    def on_run_start(self, rank: int, run: int) -> None:  # hook: caller work stream-ordered before the call
        pass

    def _start(self, g: int, st: dict) -> None:
        st["run"] += 1
        if st["run"] < len(self.args):
            self.on_run_start(g, st["run"])
        low = self.low[g]
        streams: dict[int, list] = {}
        # event semantics of stream capture: a STREAM_WAIT binds to the latest RECORD of its slot that
        # precedes it in enqueue (list) order, so event slots may be reused
        last_rec: dict[int, int] = {}
        bind: dict[int, int | None] = {}
        for i, op in enumerate(low.ops):
            streams.setdefault(op.stream, []).append(op)
            if op.op == OP_RECORD:
                last_rec[op.value] = i
            elif op.op == OP_STREAM_WAIT:
                bind[i] = last_rec.get(op.value)
        st["op_index"] = {id(op): i for i, op in enumerate(low.ops)}
        st["bind"] = bind
        st["streams"] = streams
        st["pos"] = {s: 0 for s in streams}
        st["bar_set"] = {s: False for s in streams}
        st["events"] = set()
        st["tiles"] = [{"t": t, "kseg": 0, "done": False} for t in low.tiles]
        st["memset"] = False

    def _finished(self, st: dict) -> bool:
        return (st["memset"] and all(st["pos"][s] >= len(v) for s, v in st["streams"].items())
                and all(x["done"] for x in st["tiles"]))

    def _runnable(self, g: int, st: dict) -> list:
        run = st["run"]
        par = run & 1
        rk = self.ranks[g]
        acts = []
        if not st["memset"]:
            def memset(st=st, rk=rk, par=par):
                rk.block(par ^ 1)[FICCO_FLAG_RUN_LOCAL:] = 0
                st["memset"] = True
            acts.append(memset)
        for s, ops in st["streams"].items():
            i = st["pos"][s]
            if i >= len(ops):
                continue
            op = ops[i]
            blk = rk.block(par)

            def adv(st=st, s=s):
                st["pos"][s] += 1
            if op.op == OP_COPY:
                acts.append(lambda op=op, adv=adv: (self._copy(g, run, op), adv()))
            elif op.op == OP_SIGNAL:
                n = max(1, op.value)
                acts.append(lambda op=op, blk=blk, adv=adv, n=n: (blk.__setitem__(slice(op.flag, op.flag + n),
                                                                                 0x01010101), adv()))
            elif op.op == OP_NOTIFY:
                peer_blk = self.ranks[op.peer].block(par)
                acts.append(lambda op=op, pb=peer_blk, adv=adv: (pb.__setitem__(op.flag, 1), adv()))
            elif op.op == OP_WAIT:
                if blk[op.flag] != 0:
                    acts.append(lambda op=op, blk=blk, adv=adv: (blk.__setitem__(op.flag, 0), adv()))
            elif op.op == OP_WAIT_COUNTER:
                if blk[FICCO_FLAG_COUNTERS + op.flag] >= op.value:
                    acts.append(adv)
            elif op.op == OP_BARRIER:
                w = op.flag
                if not st["bar_set"][s]:
                    def set_bytes(st=st, s=s, w=w):
                        for q in range(self.G):
                            b8 = self.ranks[q].block(par)[w:w + 4].view(np.uint8)
                            b8[g] = 1
                        st["bar_set"][s] = True
                    acts.append(set_bytes)
                else:
                    b8 = blk[w:w + 4].view(np.uint8)
                    if all(b8[q] for q in range(self.G)):
                        def done(st=st, s=s, w=w, blk=blk, adv=adv):
                            blk[w:w + 4] = 0
                            st["bar_set"][s] = False
                            adv()
                        acts.append(done)
            elif op.op == OP_RECORD:
                idx = st["op_index"][id(op)]
                acts.append(lambda idx=idx, st=st, adv=adv: (st["events"].add(idx), adv()))
            elif op.op == OP_STREAM_WAIT:
                rec = st["bind"][st["op_index"][id(op)]]
                if rec is None or rec in st["events"]:
                    acts.append(adv)
            elif op.op == OP_REDUCE_MC:
                acts.append(lambda op=op, adv=adv: (self._reduce_mc(g, run, op), adv()))
            else:
                raise AssertionError(f"unknown op {op.op}")
        num_kb = -(-self.low[g].desc.k // TILE_K)
        for x in st["tiles"]:
            if x["done"]:
                continue
            t = x["t"]
            nseg = (-(-num_kb // t.kseg)) if t.kseg else 1
            if self._tile_ready(g, run, t, x["kseg"]):
                if x["kseg"] + 1 < nseg:
                    acts.append(lambda x=x: x.__setitem__("kseg", x["kseg"] + 1))
                else:
                    d = self.low[g].desc
                    if t.mode == EPI_REDUCE:
                        blk = rk.block(par)
                        if not all(blk[d.rs_flag0 + t.chunk * d.n_recv + j] >= max(1, d.rs_target)
                                   for j in range(d.n_recv)):
                            continue
                    if t.mode == EPI_STORE_REMOTE and d.go_flag > 0 and not rk.block(par)[d.go_flag]:
                        continue  # the epilogue holds its stores until the DONE barrier passed
                    if (t.mode == EPI_STORE_SIGNAL and d.part.buf == BUF_MC and d.go_flag > 0
                            and not rk.block(par)[d.go_flag]):
                        continue  # nvls: peers read the multicast-bound partials in place
                    acts.append(lambda x=x, t=t: (self._run_tile(g, run, t), x.__setitem__("done", True)))
        return acts

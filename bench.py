"""FiCCO hot-path benchmark (driver contract: one JSON line from rank 0).

Default workload (BASELINE.json configs[1], the config the metric is quoted on):
C2 — Llama-3-8B TP/SP MLP up-projection all-gather -> GEMM, bf16, seq 8192,
per-GPU post-gather GEMM (M, N, K) = (8192, 3584 = gate||up of 14336/8, 4096).
``--workload c3`` (Llama-3-70B down-proj GEMM -> reduce-scatter, seq 16384,
(M, N, K) = (16384, 8192, 28672/G)) and ``--workload c4`` (context-parallel KV
all-gather -> QK^T, 128K context, d=128, 16384 local queries) measure the
other configs the same way.

* N = 1 (default): decomposition-only mode: this GPU plays
  rank 0 of an 8-rank job; the 7 peers' data sits in local HBM stand-in
  workspaces, so the copy engines move the same chunks (locally) and the tile
  kernel does exactly rank 0's work.
* N > 1 (torchrun): G = N real ranks over NVLink (copy-engine pulls/pushes on
  IPC-mapped workspaces), same per-GPU GEMM -> weak scaling.

A step = one overlapped op call through the public API on inputs already in
HBM. Per-step CUDA events on the compute stream, L2 flushed (256 MiB write)
between steps outside the events, all steps enqueued asynchronously between a
barrier + synchronize on each side, max over ranks. Every (schedule, comm agent)
of the design space is timed in one run, interleaved step by step (``schedules``);
the fastest is then timed again for K steps interleaved with the serialized baseline
(NCCL collective / copy-engine stand-in, then cuBLAS), so both see the same
clocks under the power cap. ``value`` = that median step time (µs, lower is
better); ``speedup_vs_serial`` = serial / value from the same interleaved run;
the ideal-overlap roofline T* sits beside them.

``--impl reference`` times the CPU restatement of the reference's path
(oracle/ficco_oracle.py — the reference itself is a pure-Python simulator with
no tensor execution) on the host cores, same metric/unit/config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AG/RS+GEMM µs & speedup vs serialized NCCL+GEMM, % ideal overlap, 2/4/8 B200"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_NOMINAL = 900e9
G_VIRTUAL = 8


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: x.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[0]) for r in self.rows if num(r[0])]
        mx = [float(r[1]) for r in self.rows if num(r[1])]
        pw = [float(r[2]) for r in self.rows if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "reasons": reasons, "samples": len(self.rows)}


def time_steps(fn, steps: int, warmup: int, flush, stream, barrier=None) -> list[float]:
    """Per-step device times (ms): CUDA events on `stream` around each step, L2 flushed between
    steps outside the events, everything enqueued asynchronously (launch latency hides behind
    the flush as in a pipelined job); barrier + synchronize on both sides of the timed steps."""
    import torch
    for _ in range(warmup):
        flush()
        fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return [a.elapsed_time(b) for a, b in evs]


def time_interleaved(fns, steps: int, warmup: int, flush, stream, barrier=None) -> list[list[float]]:
    """time_steps for several step functions ROUND-ROBIN (step i of every fn before step i+1):
    the same clocks, power-cap state and L2 state (flushed before every call) for all of them,
    so their ratio is not a drift between two separate runs."""
    import torch
    for _ in range(warmup):
        for fn in fns:
            flush()
            fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
           for _ in fns]
    for i in range(steps):
        for fn, ev in zip(fns, evs):
            flush()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return [[a.elapsed_time(b) for a, b in ev] for ev in evs]


# ------------------------------------------------------------------------------------------ workloads

class AGWorkload:
    """C2: all-gather -> GEMM (TP/SP up-projection)."""

    inplace = False
    checks_multi_rank = True  # check() needs only data every rank holds
    agent = "dma"  # comm_agent: copy engines ("dma") or SM copy kernels ("core")

    key = "c2"
    title = "C2 Llama-3-8B TP/SP MLP up-proj AG->GEMM"
    kinds = ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "uniform_fused_2d", "shard_overlap_p2p",
             "serial"]

    @staticmethod
    def shape(G):
        """Per-GPU post-gather GEMM (M, N, K): seq 8192, N = gate||up of 14336 / G (3584 at G = 8), d 4096."""
        return 8192, 2 * 14336 // G, 4096

    def __init__(self, torch, dev, G, rank, world, ops):
        self.t, self.dev, self.G, self.rank, self.world, self.ops = torch, dev, G, rank, world, ops
        self.M, self.N, self.K = self.shape(G)
        self.R = self.M // G
        # shard p from seed 1000 + p on every rank: each rank publishes shards[rank] and can check
        # the gathered result against the same global A at any N (parity_spot_check)
        self.shards = []
        for p in range(G):
            gen = torch.Generator(device=dev).manual_seed(1000 + p)
            self.shards.append((torch.rand(self.R, self.K, generator=gen, device=dev) * 2 - 1).to(torch.bfloat16))
        self.local = self.shards[rank]
        wgen = torch.Generator(device=dev).manual_seed(99)
        self.w = (torch.randn(self.N, self.K, generator=wgen, device=dev) / math.sqrt(self.K)).to(torch.bfloat16)
        self.out = torch.empty(self.M, self.N, dtype=torch.bfloat16, device=dev)
        self.gathered = torch.empty(self.M, self.K, dtype=torch.bfloat16, device=dev)
        self.flops = 2.0 * self.M * self.N * self.K
        self.comm_bytes = (G - 1) * self.R * self.K * 2

    def config(self):
        return {"M": self.M, "N": self.N, "K": self.K, "seq_len": self.M}

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_ag(grp, self.R, self.K, self.N, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_shards(low, self.shards)
        if self.inplace:  # the shard already sits in this rank's workspace slot, both parities
            for par in (0, 1):
                off = low.gather_off + par * low.gather_par + grp.rank * self.R * self.K * 2
                grp.ws_tensor(grp.rank, off, (self.R, self.K)).copy_(self.local)

    def lowered(self, grp, kind):
        return self.ops.prepare_ag(grp, self.R, self.K, self.N, kind, inplace=self.inplace, comm_agent=self.agent)[1]

    def run_plan(self, plan):
        """A raw lowered plan with this workload's call arguments (copy-program timing)."""
        plan.run(self.local, self.w, self.out)

    def step(self, grp, kind):
        agent = self.agent  # bound now: steps of both agents are interleaved
        if self.inplace:
            def fn():
                a = grp.input_slot(self.R, self.K, self.N, kind)
                self.ops.all_gather_matmul(a, self.w, kind=kind, group=grp, out=self.out, comm_agent=agent)
            return fn
        return lambda: self.ops.all_gather_matmul(self.local, self.w, kind=kind, group=grp, out=self.out,
                                                  comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.distributed.all_gather_into_tensor(self.gathered, self.local)
                t.matmul(self.gathered, self.w.T, out=self.out)
            return fn, "NCCL all_gather_into_tensor + cuBLAS"

        def fn():
            for p in range(self.G):
                self.gathered[p * self.R:(p + 1) * self.R].copy_(self.shards[p], non_blocking=True)
            t.matmul(self.gathered, self.w.T, out=self.out)
        return fn, "copy-engine gather of the 7 peer shards + cuBLAS (virtual peers)"

    def cublas(self):
        a = self.t.cat(self.shards)
        return lambda: self.t.matmul(a, self.w.T, out=self.out)

    def kernel(self, runtime):
        a = self.t.cat(self.shards)
        return lambda: runtime.gemm_bf16(a, self.w, self.out), "tensor", self.flops

    def check(self):
        rows = slice(0, 256)
        ref = self.t.cat(self.shards)[rows].float() @ self.w.float().T
        return bool(self.t.allclose(self.out[rows].float(), ref, rtol=1.6e-2, atol=1e-2))

    def e2e(self, grp, kind):
        t = self.t
        host_a = self.local.cpu().pin_memory()
        host_c = t.empty(self.M, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.local)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.all_gather_matmul(dev_a, self.w, kind=kind, group=grp, out=self.out)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.R * self.K * 2, self.M * self.N * 2

    def ideal_parts(self, peaks):
        """(T_gemm, T_comm) in µs: GEMM at the measured bf16 peak, bytes at nominal NVLink."""
        return self.flops / (peaks["bf16_tflops"] * 1e12) * 1e6, self.comm_bytes / NVLINK_NOMINAL * 1e6

    def ideal_us(self, peaks):
        return max(self.ideal_parts(peaks))

    def cpu_sample(self, orc, kind):
        sh = [s.float().cpu().numpy() for s in self.shards]
        w = self.w.float().cpu().numpy()
        frags = orc.gemm_fragments(kind, self.M, self.K, self.G, 0)
        rows_first = sum(c for rows, _ in frags[:1] for _, c in rows)
        orc.execute_ag_rank(kind, sh, w, 0, steps=1)
        t0, reps = time.perf_counter(), 0
        while reps < 5 and time.perf_counter() - t0 < 10.0:
            orc.execute_ag_rank(kind, sh, w, 0, steps=1)
            reps += 1
        per_op = (time.perf_counter() - t0) / reps * (self.M / rows_first)
        return per_op, (f"oracle execute_ag_rank({kind}): first GemmSpec ({rows_first}/{self.M} rows) x{reps}, "
                        f"scaled linearly to the full op")


class RSWorkload(AGWorkload):
    """C3: GEMM -> reduce-scatter (TP/SP down-projection)."""

    key = "c3"
    title = "C3 Llama-3-70B TP/SP down-proj GEMM->RS"
    kinds = ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d"]

    def __init__(self, torch, dev, G, rank, world, ops):
        self.t, self.dev, self.G, self.rank, self.world, self.ops = torch, dev, G, rank, world, ops
        self.M, self.N, self.K = 16384, 8192, 28672 // G
        self.R = self.M // G
        # rank g's operands from seeds 2000 + g / 3000 + g on every rank: each rank regenerates the peers'
        # partials of its own rows, which are the virtual peers' data at N = 1 and the reference the
        # parity spot check sums at any N (owner's fp32 partial + peers' bf16 partials, rank order)
        def operands(g):
            ga = torch.Generator(device=dev).manual_seed(2000 + g)
            gw = torch.Generator(device=dev).manual_seed(3000 + g)
            return ((torch.rand(self.M, self.K, generator=ga, device=dev) * 2 - 1).to(torch.bfloat16),
                    (torch.randn(self.N, self.K, generator=gw, device=dev) / math.sqrt(self.K)).to(torch.bfloat16))
        self.a, self.w = operands(rank)
        self.own = slice(rank * self.R, (rank + 1) * self.R)
        self.peer_parts = []
        for g in range(G):
            if g != rank:
                a_g, w_g = operands(g)
                self.peer_parts.append(torch.matmul(a_g[self.own], w_g.t()).to(torch.bfloat16))
                del a_g, w_g
        self.out = torch.empty(self.R, self.N, dtype=torch.bfloat16, device=dev)
        self.part = torch.empty(self.M, self.N, dtype=torch.bfloat16, device=dev)
        self.sink = torch.empty((G - 1) * self.R, self.N, dtype=torch.bfloat16, device=dev)
        self.flops = 2.0 * self.M * self.N * self.K
        self.comm_bytes = (G - 1) * self.R * self.N * 2

    def config(self):
        return {"M": self.M, "N": self.N, "K": self.K, "seq_len": self.M}

    def lowered(self, grp, kind):
        return self.ops.prepare_rs(grp, self.M, self.K, self.N, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_rs(grp, self.M, self.K, self.N, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_partials(low, self.peer_parts)

    run_plan = None  # the RS pushes wait on tile counters: no copy program runs without its tiles

    def step(self, grp, kind):
        agent = self.agent
        return lambda: self.ops.matmul_reduce_scatter(self.a, self.w, kind=kind, group=grp, out=self.out,
                                                      comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.matmul(self.a, self.w.T, out=self.part)
                t.distributed.reduce_scatter_tensor(self.out, self.part)
            return fn, "cuBLAS + NCCL reduce_scatter_tensor"
        R = self.R

        peers = t.stack(self.peer_parts)  # the received partials, contiguous like an NCCL receive buffer

        def fn():
            t.matmul(self.a, self.w.T, out=self.part)
            self.sink.copy_(self.part[R:], non_blocking=True)  # the 7 remote shards leave (copy engine)
            # one pass over the received partials (fp32 sum), then the own partial and one rounding
            acc = t.sum(peers, dim=0, dtype=t.float32)
            self.out.copy_(acc.add_(self.part[:R]))
        return fn, ("cuBLAS + copy-engine egress of 7 shards + fused fp32 reduction of the 7 received partials "
                    "and the own one (virtual peers)")

    def cublas(self):
        return lambda: self.t.matmul(self.a, self.w.T, out=self.part)

    def kernel(self, runtime):
        return lambda: runtime.gemm_bf16(self.a, self.w, self.part), "tensor", self.flops

    def check(self):
        ref = self.a[self.own].float() @ self.w.float().T
        for p in self.peer_parts:
            ref += p.float()
        return bool(self.t.allclose(self.out.float(), ref, rtol=1.6e-2, atol=3e-2))

    def e2e(self, grp, kind):
        t = self.t
        host_a = self.a.cpu().pin_memory()
        host_c = t.empty(self.R, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.a)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.matmul_reduce_scatter(dev_a, self.w, kind=kind, group=grp, out=self.out)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.M * self.K * 2, self.R * self.N * 2

    def cpu_sample(self, orc, kind):
        a = self.a[: self.R].float().cpu().numpy()
        w = self.w.float().cpu().numpy()
        t0 = time.perf_counter()
        a @ w.T
        per_op = (time.perf_counter() - t0) * self.G
        return per_op, f"numpy fp32 GEMM of one {self.R}-row chunk, scaled x{self.G} (partials of the whole op)"


class CPWorkload(AGWorkload):
    """C4: context-parallel KV all-gather -> attention scores S = Q K^T / sqrt(d)."""

    key = "c4"
    title = "C4 CP KV all-gather -> QK^T, 128K context, d=128"
    kinds = ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "shard_overlap_p2p", "serial"]

    def __init__(self, torch, dev, G, rank, world, ops):
        self.t, self.dev, self.G, self.rank, self.world, self.ops = torch, dev, G, rank, world, ops
        self.Tkv, self.Tq, self.d = 131072, 131072 // G, 128
        self.R = self.Tkv // G
        gen = torch.Generator(device=dev).manual_seed(rank)
        self.q = torch.randn(self.Tq, self.d, generator=gen, device=dev).to(torch.bfloat16)
        # K shard p from seed 1000 + p on every rank (this rank publishes shards[rank]): the score check
        # needs only the local queries and the global K, so it runs at any N
        self.shards = []
        for p in range(G):
            kgen = torch.Generator(device=dev).manual_seed(1000 + p)
            self.shards.append(torch.randn(self.R, self.d, generator=kgen, device=dev).to(torch.bfloat16))
        self.local = self.shards[rank]
        self.out = torch.empty(self.Tq, self.Tkv, dtype=torch.bfloat16, device=dev)
        self.kall = torch.empty(self.Tkv, self.d, dtype=torch.bfloat16, device=dev)
        self.scale = 1.0 / math.sqrt(self.d)
        self.flops = 2.0 * self.Tq * self.Tkv * self.d
        self.out_bytes = self.Tq * self.Tkv * 2
        self.comm_bytes = (G - 1) * self.R * self.d * 2

    def config(self):
        return {"Tkv": self.Tkv, "Tq": self.Tq, "d": self.d, "seq_len": self.Tkv}

    def lowered(self, grp, kind):
        return self.ops.prepare_cp(grp, self.Tq, self.d, self.Tkv, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_cp(grp, self.Tq, self.d, self.Tkv, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_shards(low, self.shards)

    def run_plan(self, plan):
        plan.run(self.q, self.local, self.out)

    def step(self, grp, kind):
        agent = self.agent
        return lambda: self.ops.cp_kv_all_gather_qk(self.q, self.local, kind=kind, group=grp, out=self.out,
                                                    comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.distributed.all_gather_into_tensor(self.kall, self.local)
                t.addmm(self.out, self.q, self.kall.T, beta=0, alpha=self.scale, out=self.out)
            return fn, "NCCL all_gather_into_tensor + cuBLAS (alpha = 1/sqrt(d))"

        def fn():
            for p in range(self.G):
                self.kall[p * self.R:(p + 1) * self.R].copy_(self.shards[p], non_blocking=True)
            t.addmm(self.out, self.q, self.kall.T, beta=0, alpha=self.scale, out=self.out)
        return fn, "copy-engine gather of the 7 peer K shards + cuBLAS (virtual peers)"

    def cublas(self):
        k = self.t.cat(self.shards)
        return lambda: self.t.addmm(self.out, self.q, k.T, beta=0, alpha=self.scale, out=self.out)

    def kernel(self, runtime):
        k = self.t.cat(self.shards)
        return lambda: runtime.gemm_bf16(self.q, k, self.out, alpha=self.scale), "hbm", self.out_bytes

    def check(self):
        k = self.t.cat(self.shards)
        ref = (self.q[:256].float() @ k.float().T) * self.scale
        return bool(self.t.allclose(self.out[:256].float(), ref, rtol=1.6e-2, atol=1e-2))

    def e2e(self, grp, kind):
        t = self.t
        host_q = self.q.cpu().pin_memory()
        host_k = self.local.cpu().pin_memory()
        host_s = t.empty(self.Tq, self.Tkv, dtype=t.bfloat16).pin_memory()
        dq, dk = t.empty_like(self.q), t.empty_like(self.local)

        def fn():
            dq.copy_(host_q, non_blocking=True)
            dk.copy_(host_k, non_blocking=True)
            self.ops.cp_kv_all_gather_qk(dq, dk, kind=kind, group=grp, out=self.out)
            host_s.copy_(self.out, non_blocking=True)
        return fn, (self.Tq + self.R) * self.d * 2, self.out_bytes

    def ideal_parts(self, peaks):
        t_hbm = (self.out_bytes + (self.Tq + self.Tkv) * self.d * 2) / (peaks["hbm_gbs"] * 1e9)
        t_gemm = max(self.flops / (peaks["bf16_tflops"] * 1e12), t_hbm)
        return t_gemm * 1e6, self.comm_bytes / NVLINK_NOMINAL * 1e6

    def cpu_sample(self, orc, kind):
        q = self.q[:512].float().cpu().numpy()
        k = self.t.cat(self.shards).float().cpu().numpy()
        t0 = time.perf_counter()
        (q @ k.T) * self.scale
        per_op = (time.perf_counter() - t0) * (self.Tq / 512)
        return per_op, f"numpy fp32 scores for 512 of {self.Tq} queries, scaled linearly"


class EPWorkload(AGWorkload):
    """EP all-to-all (token dispatch) -> expert GEMM: the reference corpus row g14 (Mixtral,
    data/scenarios_corpus.csv:17): per-GPU post-dispatch GEMM (M, N, K) = (147456, 28672, 4096), G = 8.
    Not a BASELINE.json config; same metric and method."""

    checks_multi_rank = False  # check() needs peers' data this rank does not hold

    key = "ep"
    title = "EP Mixtral all-to-all -> expert GEMM (corpus g14)"
    inplace = False

    def __init__(self, torch, dev, G, rank, world, ops):
        self.t, self.dev, self.G, self.rank, self.world, self.ops = torch, dev, G, rank, world, ops
        self.M, self.N, self.K = 147456, 28672, 4096
        self.R = self.M // G
        gen = torch.Generator(device=dev).manual_seed(rank)
        self.send = (torch.rand(self.M, self.K, generator=gen, device=dev) * 2 - 1).to(torch.bfloat16)
        # virtual peers' blocks addressed to this rank (peer p's block `rank`)
        self.blocks = [(torch.rand(self.R, self.K, generator=gen, device=dev) * 2 - 1).to(torch.bfloat16)
                       if p != rank else self.send[rank * self.R:(rank + 1) * self.R] for p in range(G)]
        wgen = torch.Generator(device=dev).manual_seed(100 + rank)
        self.w = (torch.randn(self.N, self.K, generator=wgen, device=dev) / math.sqrt(self.K)).to(torch.bfloat16)
        self.out = torch.empty(self.M, self.N, dtype=torch.bfloat16, device=dev)
        self.gathered = torch.empty(self.M, self.K, dtype=torch.bfloat16, device=dev)
        self.flops = 2.0 * self.M * self.N * self.K
        self.comm_bytes = (G - 1) * self.R * self.K * 2

    def lowered(self, grp, kind):
        return self.ops.prepare_a2a(grp, self.R, self.K, self.N, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_a2a(grp, self.R, self.K, self.N, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_sends(low, self.blocks)

    def run_plan(self, plan):
        plan.run(self.send, self.w, self.out)

    def step(self, grp, kind):
        agent = self.agent
        return lambda: self.ops.all_to_all_matmul(self.send, self.w, kind=kind, group=grp, out=self.out,
                                                  comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.distributed.all_to_all_single(self.gathered, self.send)
                t.matmul(self.gathered, self.w.T, out=self.out)
            return fn, "NCCL all_to_all_single + cuBLAS"

        def fn():
            for p in range(self.G):
                self.gathered[p * self.R:(p + 1) * self.R].copy_(self.blocks[p], non_blocking=True)
            t.matmul(self.gathered, self.w.T, out=self.out)
        return fn, "copy-engine dispatch of the 7 peer blocks + cuBLAS (virtual peers)"

    def cublas(self):
        a = self.t.cat(self.blocks)
        return lambda: self.t.matmul(a, self.w.T, out=self.out)

    def kernel(self, runtime):
        a = self.t.cat(self.blocks)
        return lambda: runtime.gemm_bf16(a, self.w, self.out), "tensor", self.flops

    def check(self):
        rows = slice(self.R, self.R + 256)  # peer 1's block for this rank
        ref = self.t.cat(self.blocks)[rows].float() @ self.w.float().T
        return bool(self.t.allclose(self.out[rows].float(), ref, rtol=1.6e-2, atol=1e-2))

    def e2e(self, grp, kind):
        t = self.t
        host_a = self.send.cpu().pin_memory()
        host_c = t.empty(self.M, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.send)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.all_to_all_matmul(dev_a, self.w, kind=kind, group=grp, out=self.out)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.M * self.K * 2, self.M * self.N * 2

    def cpu_sample(self, orc, kind):
        a = self.blocks[1][:1024].float().cpu().numpy()
        w = self.w.float().cpu().numpy()
        t0 = time.perf_counter()
        a @ w.T
        per_op = (time.perf_counter() - t0) * (self.M / 1024)
        return per_op, f"numpy fp32 expert GEMM of 1024 of {self.M} dispatched rows, scaled linearly"


class AG70Workload(AGWorkload):
    """C3': Llama-3-70B TP/SP MLP up-projection all-gather -> GEMM (the north star's 70B AG target):
    seq 16384, N = gate||up of 28672 / G (7168 at G = 8), d 8192."""

    key = "c3p"
    title = "C3' Llama-3-70B TP/SP MLP up-proj AG->GEMM"

    @staticmethod
    def shape(G):
        return 16384, 2 * 28672 // G, 8192


WORKLOADS = {"c2": AGWorkload, "c3": RSWorkload, "c4": CPWorkload, "ep": EPWorkload, "c3p": AG70Workload}


def our_arm(args) -> None:
    import torch
    world, rank, local = dist_env()
    # FICCO_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo — exercises the N>1 code path
    # (IPC workspaces, cross-rank protocol, max-over-ranks timing) on a one-GPU box; not a bench number
    shared = os.environ.get("FICCO_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=dev)
    from oracle import ficco_oracle as orc  # checker + CPU baseline only
    from paper_2512_10236_b200 import ops, routing, runtime
    from paper_2512_10236_b200.machines import b200_machine
    from paper_2512_10236_b200.selector import select_schedule
    runtime.load_library()

    G = args.virtual_ranks if world == 1 else world
    peaks, peaks_src = load_peaks()
    wl = WORKLOADS[args.workload](torch, dev, G, rank, world, ops)
    wl.inplace = args.input == "slot" and hasattr(wl, "shards") and args.workload in ("c2", "c3p")
    grp = ops.FiccoGroup.distributed() if world > 1 else ops.FiccoGroup.virtual_group(G, 0)
    flush_buf = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    stream = torch.cuda.current_stream()
    barrier = (lambda: torch.distributed.barrier()) if world > 1 else None

    def maxrank(ms: float) -> float:
        if world == 1:
            return ms
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # every schedule of the design space, for both comm agents (core = SM-driven transfers: AG/CP SM
    # copy kernels beside the tile kernel; RS tile epilogues storing partials straight into the owners'
    # slots), all timed in ONE interleaved run: under the power cap a box drifts by up to ~10 % within
    # a bench run (tools/switch_probe.py), so separate runs per variant would rank the drift
    sched, core, variants = {}, {}, []
    for agent in (["dma"] if args.no_core else ["dma", "core"]):
        wl.agent = agent
        for kind in (args.kinds.split(",") if args.kinds else wl.kinds):
            if agent == "core" and "error" in sched.get(kind, {"error": 1}):
                continue
            try:
                wl.prepare(grp, kind)
            except routing.PlanError as exc:
                sched[kind] = {"error": str(exc)}
                continue
            if agent == "dma":
                sched[kind] = {}
            variants.append((kind, agent, wl.step(grp, kind)))
    times = time_interleaved([fn for _, _, fn in variants], args.steps, args.warmup, flush, stream, barrier)
    grp.comm.check()
    for (kind, agent, _), ts in zip(variants, times):
        (sched if agent == "dma" else core)[kind] = {"us": maxrank(statistics.median(ts)) * 1e3}
    # the headline: the fastest (schedule, comm_agent) of the design space (serial excluded)
    cands = [(sched[k]["us"], k, "dma") for k in sched if "us" in sched[k] and k != "serial"]
    cands += [(v["us"], k, "core") for k, v in core.items() if k != "serial"]
    _, best, best_agent = min(cands)
    wl.agent = best_agent
    wl.prepare(grp, best)
    wl.step(grp, best)()
    grp.comm.check()
    parity = wl.check() if world == 1 or wl.checks_multi_rank else None

    # the headline: the best (schedule, agent) and the serialized baseline timed interleaved, K steps each
    serial_fn, serial_desc = wl.serial()
    t_best, t_serial = time_interleaved([wl.step(grp, best), serial_fn], args.steps, args.warmup, flush, stream,
                                        barrier)
    grp.comm.check()
    value = maxrank(statistics.median(t_best)) * 1e3
    serial_us = maxrank(statistics.median(t_serial)) * 1e3
    cublas_us = statistics.median(time_steps(wl.cublas(), args.steps, args.warmup, flush, stream)) * 1e3
    kern_fn, bound, work = wl.kernel(runtime)
    kern_us = statistics.median(time_steps(kern_fn, args.steps, args.warmup, flush, stream)) * 1e3
    if bound == "tensor":
        achieved, peak, unit = work / (kern_us * 1e-6) / 1e12, peaks["bf16_tflops"], "TFLOP/s"
    else:
        achieved, peak, unit = work / (kern_us * 1e-6) / 1e9, peaks["hbm_gbs"], "GB/s"

    with ClockSampler(local) as cs:  # clocks while the headline op runs back to back (~1.5 s)
        fn = wl.step(grp, best)
        t_end = time.time() + 1.5
        while time.time() < t_end:
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
    clocks = cs.summary()

    e2e_fn, h2d, d2h = wl.e2e(grp, best)
    e2e_us = maxrank(statistics.median(time_steps(e2e_fn, max(3, args.steps // 3), 3, flush, stream,
                                                  barrier))) * 1e3

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        per_op, sample = wl.cpu_sample(orc, best)
        cpu = {"value": round(per_op * 1e6, 1), "unit": "us", "cores": torch.get_num_threads(), "kind": "port",
               "sample": sample}

    b200 = b200_machine()
    sc = ops._scenario(wl.key, *((wl.M, wl.N, wl.K) if hasattr(wl, "M") else (wl.Tkv, wl.Tq, wl.d)), G)
    selector_kind = select_schedule(sc, b200.machine, b200.t_ref).value
    value_sequential = (core if best_agent == "core" else sched)[best]["us"]
    low = wl.lowered(grp, best)
    core_copies = sum(op.op == runtime.OP_COPY and op.src_buf == runtime.BUF_WS and op.dst_buf == runtime.BUF_WS
                      for op in low.ops) if low.desc.hints & runtime.FICCO_HINT_CORE_COPIES else 0
    t_star = wl.ideal_us(peaks)
    t_fill = max(wl.ideal_parts(peaks)) + min(wl.ideal_parts(peaks)) / G  # the reference's pipelined ideal
    # the copy program alone, replayed from its CUDA graph (empty tile list): measured transfer rate
    copy_gbps = None
    if world == 1 and wl.run_plan is not None:
        copy_low = wl.lowered(grp, best)
        copy_plan = runtime.Plan(grp.comm, copy_low.desc, list(copy_low.ops), [])
        try:
            copy_us = statistics.median(time_steps(lambda: wl.run_plan(copy_plan), args.steps, args.warmup, flush,
                                                   stream)) * 1e3
            copy_gbps = round(wl.comm_bytes / (copy_us * 1e-6) / 1e9, 1)
        finally:
            copy_plan.close()
    if rank == 0:
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", f"r01_ncu_traffic_{wl.key}.json")) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            pass
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(value / 1e3, 5), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded uniform/normal inputs of the config's shapes)",
            "config": dict(workload=wl.title, ranks=G, virtual_peers=world == 1, schedule=best,
                           comm_agent=best_agent,
                           input="symmetric slot (zero-copy publish)" if wl.inplace else "tensor copied in",
                           selector_schedule=selector_kind, l2="flushed (256 MiB write) between timed steps",
                           **wl.config()),
            "speedup_vs_serial": round(serial_us / value, 4), "serial_us": round(serial_us, 2),
            "timing": "schedules: every (kind, agent) variant interleaved step by step in one run; value and "
                      "serial_us: the best variant and the serialized baseline interleaved in a second run "
                      "(the box drifts up to ~10 % between runs under the power cap)",
            "value_sequential": round(value_sequential, 2),
            "serial_baseline": serial_desc, "cublas_gemm_us": round(cublas_us, 2),
            "ideal_overlap_us": round(t_star, 2), "pct_ideal_overlap": round(t_star / value, 4),
            "ideal_overlap_fill_us": round(t_fill, 2), "pct_ideal_overlap_fill": round(t_fill / value, 4),
            "copy_program_GBps": copy_gbps,
            "schedules": {k: ({"us": round(v["us"], 2)} if "us" in v else v) for k, v in sched.items()},
            "schedules_comm_agent_core": {k: {"us": round(v["us"], 2)} for k, v in core.items()},
            "parity_spot_check": parity,
            "roofline": {"bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "frac_sustained": (round(achieved / peaks["bf16_tflops_sustained"], 4)
                                            if bound == "tensor" and "bf16_tflops_sustained" in peaks else None),
                         "kernel": "ficco::tile_gemm_kernel (flag-free plain GEMM of the op's shape, same kernel)",
                         "kernel_us": round(kern_us, 2),
                         "peak_source": f"MEASURED_PEAKS.json ({peaks_src}; burst figure, kernel timed alone)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_us, 2), "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps * (1 + core_copies),
            "clocks": clocks,
        }))
    grp.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def reference_arm(args) -> None:
    """CPU restatement of the reference's path (the oracle port) on the host cores, C2 config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    from oracle import ficco_oracle as orc
    G, M, N, K = G_VIRTUAL, 8192, 3584, 4096
    R = M // G
    shards = [orc.seeded_inputs(0, p, (R, K)) for p in range(G)]
    w = orc.seeded_inputs(0, 99, (N, K), "normal")
    kind = "uniform_fused_1d"
    frags = orc.gemm_fragments(kind, M, K, G, 0)
    rows_first = sum(c for rows, _ in frags[:1] for _, c in rows)
    scale = M / rows_first
    for _ in range(max(1, min(args.warmup, 2))):
        orc.execute_ag_rank(kind, shards, w, 0, steps=1)
    times = []
    for _ in range(max(1, min(args.steps, 20))):
        t0 = time.perf_counter()
        orc.execute_ag_rank(kind, shards, w, 0, steps=1)
        times.append((time.perf_counter() - t0) * scale)
    us = statistics.median(times) * 1e6
    sample = (f"oracle port (numpy fp32 BLAS) of rank 0's {kind} AG->GEMM: first step ({rows_first}/{M} rows) "
              f"per timed step, scaled x{scale:g}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": "us", "n_gpus": world,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": round(us / 1e3, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": AGWorkload.title, "M": M, "N": N, "K": K, "ranks": G, "schedule": kind},
        "cpu_baseline": {"value": round(us, 1), "unit": "us", "cores": torch.get_num_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(us, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ficco", choices=["ficco", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--kinds", default="", help="comma-separated subset of schedules")
    ap.add_argument("--virtual-ranks", type=int, default=G_VIRTUAL,
                    help="N=1 only: the job size G this GPU plays rank 0 of (C3 is quoted at G = 2, 4 and 8)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-core", action="store_true", help="skip the comm_agent=core (SM copies) comparison")
    ap.add_argument("--input", default="slot", choices=["slot", "copy"],
                    help="slot: the A shard is produced in the group's symmetric input slot (zero-copy publish, "
                         "FiccoGroup.input_slot); copy: an ordinary tensor copied in by the op")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()

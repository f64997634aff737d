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
# one hardware queue per stream (see paper_2512_10236_b200/__init__.py): must precede the first CUDA call
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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

    @staticmethod
    def merge(*samplers):
        m = ClockSampler(-1)
        for smp in samplers:
            m.rows += smp.rows
        return m.summary()

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


def coll_backend() -> str:
    """The collective library behind torch.distributed here: NCCL, or gloo in the shared-GPU plumbing check."""
    import torch
    return "NCCL" if torch.distributed.get_backend() == "nccl" else "gloo (shared-GPU plumbing check)"


def time_interleaved(fns, steps: int, warmup: int, flush, stream, barrier=None, starts=None) -> list[list[float]]:
    """time_steps for several step functions ROUND-ROBIN (step i of every fn before step i+1):
    the same clocks, power-cap state and L2 state (flushed before every call) for all of them,
    so their ratio is not a drift between two separate runs. ``starts`` (a list) receives the
    (start, end) events of the first function's timed steps."""
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
    if starts is not None:
        starts.extend(evs[0])
    return [[a.elapsed_time(b) for a, b in ev] for ev in evs]


# ------------------------------------------------------------------------------------------ workloads

class AGWorkload:
    """C2: all-gather -> GEMM (TP/SP up-projection)."""

    inplace = False
    checks_multi_rank = True  # check() needs only data every rank holds
    agent = "dma"  # comm_agent: copy engines ("dma") or SM copy kernels ("core")

    key = "c2"
    op = "ag"
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

    @classmethod
    def op_shape(cls, G):
        """The scenario (M, N, K) the selector sees (the reference's per-GPU post-gather GEMM)."""
        return cls.shape(G)

    @classmethod
    def shape_config(cls, G):
        m, n, k = cls.shape(G)
        return {"M": m, "N": n, "K": k, "seq_len": m}

    def plan_for(self, grp, kind, agent):
        return self.ops.prepare_ag(grp, self.R, self.K, self.N, kind, inplace=self.inplace, comm_agent=agent)[0]

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

    def step(self, grp, kind, agent="self"):
        agent = self.agent if agent == "self" else agent  # bound now: steps of both agents are interleaved
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
            return fn, f"{coll_backend()} all_gather_into_tensor + cuBLAS"

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

    def e2e(self, grp, kind, agent=None):
        t = self.t
        host_a = self.local.cpu().pin_memory()
        host_c = t.empty(self.M, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.local)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.all_gather_matmul(dev_a, self.w, kind=kind, group=grp, out=self.out, comm_agent=agent)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.R * self.K * 2, self.M * self.N * 2

    def ideal_parts(self, peaks):
        """(T_gemm, T_comm) in µs: GEMM at the measured bf16 peak, bytes at nominal NVLink."""
        return self.flops / (peaks["bf16_tflops"] * 1e12) * 1e6, self.comm_bytes / NVLINK_NOMINAL * 1e6

    def ideal_us(self, peaks):
        return max(self.ideal_parts(peaks))

    def cpu_op(self, orc, kind):
        """Rank `rank`'s whole op on the host cores (oracle port): route + every GemmSpec fragment.
        Returns (fn, sample description, fraction of the op one call does)."""
        sh = [s.float().cpu().numpy() for s in self.shards]
        w = self.w.float().cpu().numpy()
        return (lambda: orc.execute_ag_rank(kind, sh, w, self.rank),
                f"oracle execute_ag_rank({kind}), rank {self.rank}'s whole op: the plan's routing of the {self.G} "
                f"shards + every GemmSpec fragment, fp32 numpy BLAS", 1.0)


class RSWorkload(AGWorkload):
    """C3: GEMM -> reduce-scatter (TP/SP down-projection)."""

    key = "c3"
    op = "rs"
    title = "C3 Llama-3-70B TP/SP down-proj GEMM->RS"
    # every executable RS adjoint (lowering.rs_pieces): the fine-grain kinds, the N-block 2D adjoint,
    # the reversed shard ring and the serial push-after-GEMM
    kinds = ["uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "uniform_fused_2d", "shard_overlap_p2p",
             "serial"]

    def __init__(self, torch, dev, G, rank, world, ops):
        self.t, self.dev, self.G, self.rank, self.world, self.ops = torch, dev, G, rank, world, ops
        self.M, self.N, self.K = self.shape(G)
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
                if dev.type == "cpu":  # reference arm: bf16 GEMMs on the host are slow; same values via fp32
                    self.peer_parts.append(torch.matmul(a_g[self.own].float(), w_g.float().t()).to(torch.bfloat16))
                else:
                    self.peer_parts.append(torch.matmul(a_g[self.own], w_g.t()).to(torch.bfloat16))
                del a_g, w_g
        self.out = torch.empty(self.R, self.N, dtype=torch.bfloat16, device=dev)
        self.part = torch.empty(self.M, self.N, dtype=torch.bfloat16, device=dev)
        self.sink = torch.empty((G - 1) * self.R, self.N, dtype=torch.bfloat16, device=dev)
        self.flops = 2.0 * self.M * self.N * self.K
        self.comm_bytes = (G - 1) * self.R * self.N * 2

    @staticmethod
    def shape(G):
        """Per-GPU GEMM (M, N, K) of the down-projection: seq 16384, d 8192, K = 28672 / G."""
        return 16384, 8192, 28672 // G

    def plan_for(self, grp, kind, agent):
        return self.ops.prepare_rs(grp, self.M, self.K, self.N, kind, comm_agent=agent)[0]

    def lowered(self, grp, kind):
        return self.ops.prepare_rs(grp, self.M, self.K, self.N, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_rs(grp, self.M, self.K, self.N, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_partials(low, self.peer_parts)

    run_plan = None  # the RS pushes wait on tile counters: no copy program runs without its tiles

    def step(self, grp, kind, agent="self"):
        agent = self.agent if agent == "self" else agent
        return lambda: self.ops.matmul_reduce_scatter(self.a, self.w, kind=kind, group=grp, out=self.out,
                                                      comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.matmul(self.a, self.w.T, out=self.part)
                t.distributed.reduce_scatter_tensor(self.out, self.part)
            return fn, f"cuBLAS + {coll_backend()} reduce_scatter_tensor"
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

    def e2e(self, grp, kind, agent=None):
        t = self.t
        host_a = self.a.cpu().pin_memory()
        host_c = t.empty(self.R, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.a)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.matmul_reduce_scatter(dev_a, self.w, kind=kind, group=grp, out=self.out, comm_agent=agent)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.M * self.K * 2, self.R * self.N * 2

    def cpu_op(self, orc, kind):
        a = self.a.float().cpu().numpy()
        w = self.w.float().cpu().numpy()
        peers = [p.float().cpu().numpy() for p in self.peer_parts]
        return (lambda: orc.execute_rs_rank(a, w, peers, self.rank),
                f"oracle execute_rs_rank, rank {self.rank}'s whole op: the {self.M}-row partial GEMM + the reduction "
                f"of its {self.R} rows with the {self.G - 1} received partials, fp32 numpy BLAS", 1.0)


class CPWorkload(AGWorkload):
    """C4: context-parallel KV all-gather -> attention scores S = Q K^T / sqrt(d)."""

    key = "c4"
    op = "cp"
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

    @staticmethod
    def op_shape(G):
        """Scenario view: M = Tkv gathered kv tokens, N = Tq local queries, K = d."""
        return 131072, 131072 // G, 128

    @classmethod
    def shape_config(cls, G):
        tkv, tq, d = cls.op_shape(G)
        return {"Tkv": tkv, "Tq": tq, "d": d, "seq_len": tkv}

    def plan_for(self, grp, kind, agent):
        return self.ops.prepare_cp(grp, self.Tq, self.d, self.Tkv, kind, comm_agent=agent, inplace=self.inplace)[0]

    def lowered(self, grp, kind):
        return self.ops.prepare_cp(grp, self.Tq, self.d, self.Tkv, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_cp(grp, self.Tq, self.d, self.Tkv, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_shards(low, self.shards)
        if self.inplace:  # the K shard already sits in this rank's workspace slot, both parities
            for par in (0, 1):
                off = low.gather_off + par * low.gather_par + grp.rank * self.R * self.d * 2
                grp.ws_tensor(grp.rank, off, (self.R, self.d)).copy_(self.local)

    def run_plan(self, plan):
        plan.run(self.q, self.local, self.out)

    def step(self, grp, kind, agent="self"):
        agent = self.agent if agent == "self" else agent
        if self.inplace:
            def fn():
                k = grp.kv_slot(self.Tq, self.d, self.Tkv, kind)
                self.ops.cp_kv_all_gather_qk(self.q, k, kind=kind, group=grp, out=self.out, comm_agent=agent)
            return fn
        return lambda: self.ops.cp_kv_all_gather_qk(self.q, self.local, kind=kind, group=grp, out=self.out,
                                                    comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.distributed.all_gather_into_tensor(self.kall, self.local)
                t.addmm(self.out, self.q, self.kall.T, beta=0, alpha=self.scale, out=self.out)
            return fn, f"{coll_backend()} all_gather_into_tensor + cuBLAS (alpha = 1/sqrt(d))"

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

    def e2e(self, grp, kind, agent=None):
        t = self.t
        host_q = self.q.cpu().pin_memory()
        host_k = self.local.cpu().pin_memory()
        host_s = t.empty(self.Tq, self.Tkv, dtype=t.bfloat16).pin_memory()
        dq, dk = t.empty_like(self.q), t.empty_like(self.local)

        def fn():
            dq.copy_(host_q, non_blocking=True)
            dk.copy_(host_k, non_blocking=True)
            self.ops.cp_kv_all_gather_qk(dq, dk, kind=kind, group=grp, out=self.out, comm_agent=agent)
            host_s.copy_(self.out, non_blocking=True)
        return fn, (self.Tq + self.R) * self.d * 2, self.out_bytes

    def ideal_parts(self, peaks):
        t_hbm = (self.out_bytes + (self.Tq + self.Tkv) * self.d * 2) / (peaks["hbm_gbs"] * 1e9)
        t_gemm = max(self.flops / (peaks["bf16_tflops"] * 1e12), t_hbm)
        return t_gemm * 1e6, self.comm_bytes / NVLINK_NOMINAL * 1e6

    def cpu_op(self, orc, kind):
        q = self.q.float().cpu().numpy()
        ks = [k.float().cpu().numpy() for k in self.shards]
        import numpy as np
        sink = np.empty((self.Tq, self.R), dtype=np.float32)
        return (lambda: orc.execute_cp_qk_rank(kind, q, ks, self.scale, self.rank, sink),
                f"oracle execute_cp_qk_rank({kind}), rank {self.rank}'s whole op: K gathered by the plan's routing, "
                f"scores of every fragment (fp32 numpy BLAS) into a [{self.Tq}, {self.R}] staging block (the "
                f"8.6 GB fp32 score matrix is not kept)", 1.0)


class EPWorkload(AGWorkload):
    """EP all-to-all (token dispatch) -> expert GEMM: the reference corpus row g14 (Mixtral,
    data/scenarios_corpus.csv:17): per-GPU post-dispatch GEMM (M, N, K) = (147456, 28672, 4096), G = 8.
    Not a BASELINE.json config; same metric and method."""

    checks_multi_rank = False  # check() needs peers' data this rank does not hold

    key = "ep"
    op = "a2a"
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

    @staticmethod
    def shape(G):
        return 147456, 28672, 4096

    def plan_for(self, grp, kind, agent):
        return self.ops.prepare_a2a(grp, self.R, self.K, self.N, kind, comm_agent=agent)[0]

    def lowered(self, grp, kind):
        return self.ops.prepare_a2a(grp, self.R, self.K, self.N, kind, comm_agent=self.agent)[1]

    def prepare(self, grp, kind):
        _, low, _ = self.ops.prepare_a2a(grp, self.R, self.K, self.N, kind, comm_agent=self.agent)
        if grp.virtual:
            grp.load_peer_sends(low, self.blocks)

    def run_plan(self, plan):
        plan.run(self.send, self.w, self.out)

    def step(self, grp, kind, agent="self"):
        agent = self.agent if agent == "self" else agent
        return lambda: self.ops.all_to_all_matmul(self.send, self.w, kind=kind, group=grp, out=self.out,
                                                  comm_agent=agent)

    def serial(self):
        t = self.t
        if self.world > 1:
            def fn():
                t.distributed.all_to_all_single(self.gathered, self.send)
                t.matmul(self.gathered, self.w.T, out=self.out)
            return fn, f"{coll_backend()} all_to_all_single + cuBLAS"

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

    def e2e(self, grp, kind, agent=None):
        t = self.t
        host_a = self.send.cpu().pin_memory()
        host_c = t.empty(self.M, self.N, dtype=t.bfloat16).pin_memory()
        dev_a = t.empty_like(self.send)

        def fn():
            dev_a.copy_(host_a, non_blocking=True)
            self.ops.all_to_all_matmul(dev_a, self.w, kind=kind, group=grp, out=self.out, comm_agent=agent)
            host_c.copy_(self.out, non_blocking=True)
        return fn, self.M * self.K * 2, self.M * self.N * 2

    def cpu_op(self, orc, kind):
        import numpy as np
        blocks = [b.float().cpu().numpy() for b in self.blocks]
        w = self.w.float().cpu().numpy()
        sink = np.empty((self.R, self.N), dtype=np.float32)
        return (lambda: orc.execute_a2a_rank(kind, blocks, w, self.rank, sink),
                f"oracle execute_a2a_rank({kind}), rank {self.rank}'s whole op: the {self.G} dispatched blocks "
                f"routed by the plan, every GemmSpec fragment (~35 TFLOP, fp32 numpy BLAS) into a [{self.R}, "
                f"{self.N}] staging block (the 17 GB fp32 output is not kept)", 1.0)


class AG70Workload(AGWorkload):
    """C3': Llama-3-70B TP/SP MLP up-projection all-gather -> GEMM (the north star's 70B AG target):
    seq 16384, N = gate||up of 28672 / G (7168 at G = 8), d 8192."""

    key = "c3p"
    title = "C3' Llama-3-70B TP/SP MLP up-proj AG->GEMM"

    @staticmethod
    def shape(G):
        return 16384, 2 * 28672 // G, 8192


class C1Workload(AGWorkload):
    """C1 (BASELINE.json configs[0]): the reference's CPU-runnable case, all-gather -> GEMM at
    M = N = K = 4096 with 4 ranks. The oracle (the CPU baseline here) computes it in fp32, the GPU path in
    bf16; the selector picks uniform_fused_2d (M <= K, heuristic.py:35)."""

    key = "c1"
    title = "C1 AG->GEMM 4096^3, 4 ranks (BASELINE configs[0])"
    default_ranks = 4

    @staticmethod
    def shape(G):
        return 4096, 4096, 4096


WORKLOADS = {"c1": C1Workload, "c2": AGWorkload, "c3": RSWorkload, "c4": CPWorkload, "ep": EPWorkload,
             "c3p": AG70Workload}


def job_ranks(args) -> int:
    """G of the N = 1 decomposition-only run: --virtual-ranks, else the workload's own (C1: 4), else 8."""
    return args.virtual_ranks or getattr(WORKLOADS[args.workload], "default_ranks", G_VIRTUAL)


def headline_choice(workload: str, G: int, args) -> tuple[str, str]:
    """The (schedule, comm_agent) the public API picks for this workload with no overrides: the
    heuristic selector (selector.select_schedule == the reference's heuristic.py:25-43, pinned by
    tests/golden/selector.json) on the B200 machine file, and the machine file's comm_agent
    (machines.py:48). Pure host computation: the reference arm derives the same config."""
    from paper_2512_10236_b200 import ops
    m, n, k = WORKLOADS[workload].op_shape(G)
    kind = args.kind or ops.choose_kind(ops._scenario(workload, m, n, k, G), None).value
    agent = args.agent or ops.default_agent(WORKLOADS[workload].op)
    return kind, agent


def workload_config(args, world: int) -> dict:
    """The JSON line's ``config`` (identical in both arms)."""
    cls = WORKLOADS[args.workload]
    G = job_ranks(args) if world == 1 else world
    kind, agent = headline_choice(args.workload, G, args)
    slot = args.input == "slot" and args.workload in ("c1", "c2", "c3p", "c4")
    return dict(workload=cls.title, ranks=G, virtual_peers=world == 1, schedule=kind, comm_agent=agent,
                schedule_source=("--kind/--agent override" if (args.kind or args.agent) else
                                 "public API default: select_schedule on the B200 machine file; "
                                 "ops.default_agent(op)"),
                input="symmetric slot (zero-copy publish)" if slot else "tensor copied in",
                l2="flushed (256 MiB write) between timed steps", **cls.shape_config(G))


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info() if i.get("user_api") == "blas")
    except Exception:
        return os.cpu_count() or 1


def time_cpu(fn, reps: int, warmup: int = 1, budget_s: float = 30.0) -> list[float]:
    """Wall-clock seconds per call of a host-side function (warm-up calls untimed)."""
    for _ in range(warmup):
        fn()
    out = []
    t_end = time.perf_counter() + budget_s
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        out.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return out


def traffic_for(key: str, G: int, kind: str, agent: str):
    """DRAM bytes per launch of the op's tile kernel from a committed ncu capture of exactly this
    (workload, G, schedule, agent) — profiles/r02_ncu_traffic_<key>_g<G>_<kind>_<agent>.json — else None."""
    path = os.path.join(ROOT, "profiles", f"r02_ncu_traffic_{key}_g{G}_{kind}_{agent}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


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
    runtime.load_library()

    G = job_ranks(args) if world == 1 else world
    peaks, peaks_src = load_peaks()
    config = workload_config(args, world)
    best, best_agent = config["schedule"], config["comm_agent"]
    api_kind = args.kind or None   # None: the op call itself selects (the headline is the public API default)
    api_agent = args.agent or None
    wl = WORKLOADS[args.workload](torch, dev, G, rank, world, ops)
    wl.inplace = config["input"].startswith("symmetric")
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

    sampler = ClockSampler(local)
    sampler.__enter__()  # clocks + throttle reasons sampled from here to the end of the timed regions

    # (1) every schedule of the design space for both comm agents (core = SM-driven transfers: AG/CP SM
    # copy kernels beside the tile kernel; RS tile epilogues storing partials straight into the owners'
    # slots), all timed in ONE interleaved run: under the power cap a box drifts by up to ~10 % within
    # a bench run (tools/switch_probe.py), so separate runs per variant would rank the drift
    sched, core, variants = {}, {}, []
    if not args.headline_only:
        for agent in (["dma"] if args.no_core else ["dma", "core"]):
            wl.agent = agent
            for kind in (args.kinds.split(",") if args.kinds else wl.kinds):
                try:
                    wl.prepare(grp, kind)
                except routing.PlanError as exc:
                    (sched if agent == "dma" else core)[kind] = {"error": str(exc)}
                    continue
                variants.append((kind, agent, wl.step(grp, kind)))
        times = time_interleaved([fn for _, _, fn in variants], args.steps, args.warmup, flush, stream, barrier)
        grp.comm.check()
        for (kind, agent, _), ts in zip(variants, times):
            (sched if agent == "dma" else core)[kind] = {"us": maxrank(statistics.median(ts)) * 1e3}

    # (2) the headline: the public API call with no schedule / agent overrides (kind=None: the selector
    # picks; comm_agent=None: the machine file's agent), interleaved step by step with the serialized
    # baseline, cuBLAS on the same GEMM and our tile kernel as a plain GEMM (same clocks for all four).
    # The op's tile kernel is timed in-op: an event recorded right behind it on the launch stream.
    wl.agent = best_agent
    wl.prepare(grp, best)
    plan = wl.plan_for(grp, best, best_agent)
    op_fn = wl.step(grp, api_kind, api_agent)
    op_fn()
    torch.cuda.synchronize()
    grp.comm.check()
    parity = wl.check() if world == 1 or wl.checks_multi_rank else None
    kev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + args.warmup)]
    for e in kev:
        e.record(stream)  # materialise the CUDA events (their handles go to the library)
    torch.cuda.synchronize()
    k_i = [0]

    def op_timed():
        plan.set_kernel_event(kev[k_i[0] % len(kev)])
        k_i[0] += 1
        op_fn()

    serial_fn, serial_desc = wl.serial()
    kern_fn, bound, work = wl.kernel(runtime)
    fns = [op_timed, serial_fn, wl.cublas(), kern_fn]
    # the executor's own serial schedule (every transfer, then the same tile kernel as one GEMM): the
    # speed-up over it is the overlap alone, without our GEMM's edge over cuBLAS
    own_serial = None
    if "serial" in wl.kinds:
        try:
            wl.agent = best_agent
            wl.prepare(grp, "serial")
            own_serial = wl.step(grp, "serial", best_agent)
            fns.append(own_serial)
        except routing.PlanError:
            own_serial = None
        wl.agent = best_agent
        wl.prepare(grp, best)
    ev_starts = []
    times = time_interleaved(fns, args.steps, args.warmup, flush, stream, barrier, starts=ev_starts)
    t_op, t_serial, t_cublas, t_kern = times[:4]
    own_serial_us = maxrank(statistics.median(times[4])) * 1e3 if own_serial else None
    plan.set_kernel_event(None)
    grp.comm.check()
    # kernel durations: step start event (recorded before the op's launches) -> event behind the kernel
    kern_in_op = [ev_starts[i][0].elapsed_time(kev[args.warmup + i]) for i in range(args.steps)]
    value = maxrank(statistics.median(t_op)) * 1e3
    serial_us = maxrank(statistics.median(t_serial)) * 1e3
    cublas_us = maxrank(statistics.median(t_cublas)) * 1e3
    kern_alone_us = maxrank(statistics.median(t_kern)) * 1e3
    kern_op_us = maxrank(statistics.median(kern_in_op)) * 1e3

    with ClockSampler(local) as cs_loop:  # the headline op back to back (~1.5 s) so the sampler sees load
        t_end = time.time() + 1.5
        while time.time() < t_end:
            for _ in range(10):
                op_fn()
            torch.cuda.synchronize()
    sampler.__exit__(None, None, None)
    clocks = ClockSampler.merge(sampler, cs_loop)

    e2e_fn, h2d, d2h = wl.e2e(grp, api_kind, api_agent)
    e2e_us = maxrank(statistics.median(time_steps(e2e_fn, max(3, args.steps // 2), 3, flush, stream,
                                                  barrier))) * 1e3

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        fn, sample, frac = wl.cpu_op(orc, best)
        ts = time_cpu(fn, reps=3, warmup=1, budget_s=20.0)
        cpu = {"value": round(statistics.median(ts) / frac * 1e6, 1), "unit": "us", "cores": blas_threads(),
               "kind": "port", "sample": f"{sample}; median of {len(ts)} timed calls after 1 warm-up"}

    low = wl.lowered(grp, best)
    core_copies = sum(op.op == runtime.OP_COPY and op.src_buf == runtime.BUF_WS and op.dst_buf == runtime.BUF_WS
                      for op in low.ops) if low.desc.hints & runtime.FICCO_HINT_CORE_COPIES else 0
    t_star = wl.ideal_us(peaks)
    t_fill = max(wl.ideal_parts(peaks)) + min(wl.ideal_parts(peaks)) / G  # the reference's pipelined ideal
    # the copy program alone, replayed from its CUDA graph (empty tile list): measured transfer rate
    copy_gbps = None
    if world == 1 and wl.run_plan is not None:
        copy_plan = runtime.Plan(grp.comm, low.desc, list(low.ops), [])
        try:
            copy_us = statistics.median(time_steps(lambda: wl.run_plan(copy_plan), args.steps, args.warmup, flush,
                                                   stream)) * 1e3
            copy_gbps = round(wl.comm_bytes / (copy_us * 1e-6) / 1e9, 1)
        finally:
            copy_plan.close()
    cands = [(v["us"], k, "dma") for k, v in sched.items() if "us" in v and k != "serial"]
    cands += [(v["us"], k, "core") for k, v in core.items() if "us" in v and k != "serial"]
    fastest = min(cands) if cands else None
    if bound == "tensor":
        unit, peak, scale = "TFLOP/s", peaks["bf16_tflops"], 1e12
    else:
        unit, peak, scale = "GB/s", peaks["hbm_gbs"], 1e9
    achieved = work / (kern_op_us * 1e-6) / scale
    ref_us = (sched if best_agent == "dma" else core).get(best, {}).get("us")

    def table_entry(v):
        if "us" not in v:
            return v
        e = {"us": round(v["us"], 2)}
        if ref_us:
            e["vs_api_default"] = round(v["us"] / ref_us, 4)
        return e

    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(value, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(value / 1e3, 5), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded uniform/normal inputs of the config's shapes)",
            "config": config,
            "speedup_vs_serial": round(serial_us / value, 4), "serial_us": round(serial_us, 2),
            "serial_baseline": serial_desc,
            "speedup_vs_own_serial": round(own_serial_us / value, 4) if own_serial_us else None,
            "own_serial_us": round(own_serial_us, 2) if own_serial_us else None,
            "own_serial_baseline": ("this executor's serial schedule (all transfers, then the same tile kernel "
                                    "as one GEMM), interleaved with the headline" if own_serial_us else None),
            "timing": "value: median of the public API op (no schedule/agent override), interleaved step by step "
                      "with the serialized baseline, cuBLAS and the plain tile GEMM (L2 flushed before each call); "
                      "schedules: every (kind, agent) variant interleaved in an earlier run",
            "cublas_gemm_us": round(cublas_us, 2),
            "ideal_overlap_us": round(t_star, 2), "pct_ideal_overlap": round(t_star / value, 4),
            "ideal_overlap_fill_us": round(t_fill, 2), "pct_ideal_overlap_fill": round(t_fill / value, 4),
            "copy_program_GBps": copy_gbps,
            "fastest_variant": ({"schedule": fastest[1], "comm_agent": fastest[2], "us": round(fastest[0], 2)}
                                if fastest else None),
            "schedules": {k: table_entry(v) for k, v in sched.items()},
            "schedules_comm_agent_core": {k: table_entry(v) for k, v in core.items()},
            "schedules_note": "one interleaved run of every variant, before the headline run; absolute times carry "
                              "that run's power-cap state (the mix of variants sets the clocks), so compare "
                              "variants through vs_api_default (variant / the API-default variant, same run)",
            "parity_spot_check": parity,
            "roofline": {"bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                         "frac": round(achieved / peak, 4), "traffic": traffic_for(wl.key, G, best, best_agent),
                         "kernel": f"ficco::tile_gemm_kernel inside the {best}/{best_agent} op: median in-op duration "
                                   f"over the timed steps (CUDA events on the launch stream: step start -> event "
                                   f"recorded behind the kernel)",
                         "kernel_us": round(kern_op_us, 2),
                         "work_per_launch": work, "work_unit": "flop" if bound == "tensor" else "byte",
                         "op_frac": round(work / (value * 1e-6) / scale / peak, 4),
                         "kernel_alone_us": round(kern_alone_us, 2),
                         "kernel_alone_frac": round(work / (kern_alone_us * 1e-6) / scale / peak, 4),
                         "frac_sustained": (round(achieved / peaks["bf16_tflops_sustained"], 4)
                                            if bound == "tensor" and "bf16_tflops_sustained" in peaks else None),
                         "peak_source": f"MEASURED_PEAKS.json ({peaks_src}; burst figure)"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_us, 2), "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps * (1 + core_copies),
            "clocks": clocks,
        }))
    grp.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def reference_simulator_us(workload: str, G: int, budget_s: float = 3.0):
    """The reference's own CPU path for this config, from the unmodified install in baseline/_ref:
    build_plan + simulate (every executable kind) + select_schedule (planner.py:409, engine.py:117,
    heuristic.py:25) on the B200 machine file, 1 host thread. Returns (µs per pass, note) or (None, why)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "overlap_sim")):
        return None, "baseline/_ref not installed"
    sys.path.insert(0, ref)
    try:
        from overlap_sim import core, engine, heuristic, lossmodel, machines, planner
        with open(os.path.join(ROOT, "paper_2512_10236_b200", "data", "machine_b200.json")) as f:
            spec = machines.machine_spec_from_dict(json.load(f))
        model = lossmodel.default_calibration()
        m, n, k = WORKLOADS[workload].op_shape(G)
        sc = core.Scenario(name=workload, parallelism=core.Parallelism.SP_TP, model="bench",
                           gemm=core.GemmShape(m, n, k, 2), collective=core.Collective.ALL_GATHER, n_gpus=G)
        topo = spec.topo if spec.topo.n_gpus == G else type(spec.topo)(
            kind=spec.topo.kind, n_gpus=G, link_bw=spec.topo.link_bw, nic_bw=spec.topo.nic_bw,
            latency=spec.topo.latency)

        def one_pass():
            heuristic.select_schedule(sc, spec.machine, spec.t_ref)
            for kind in planner.supported_kinds(sc):
                engine.simulate(planner.build_plan(sc, kind, topo), spec.machine, topo, model)

        ts = time_cpu(one_pass, reps=1000, warmup=1, budget_s=budget_s)
        return statistics.median(ts) * 1e6, (f"overlap_sim {G}-rank {workload} scenario: select_schedule + "
                                             f"build_plan/simulate of every supported kind, {len(ts)} passes")
    except Exception as exc:  # pragma: no cover - reported, never fatal
        return None, f"reference simulator failed: {exc!r}"
    finally:
        sys.path.remove(ref)


def reference_arm(args) -> None:
    """The reference's CPU implementation of the path on the host cores, on our arm's config.

    The reference (overlap_sim) is a simulator: it plans and prices schedules but moves no tensor
    data, so the executable CPU path is the oracle port (oracle/ficco_oracle.py, which
    restates the reference's routing and is pinned to its plans): each step runs rank 0's WHOLE op of
    the config's schedule (no sampling or scaling; numpy fp32 BLAS on all host threads). The
    reference's own planning/pricing path (baseline/_ref) is timed beside it.
    """
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    from oracle import ficco_oracle as orc
    config = workload_config(args, world)
    G = config["ranks"]
    wl = WORKLOADS[args.workload](torch, torch.device("cpu"), G, 0, 1, None)
    fn, sample, frac = wl.cpu_op(orc, config["schedule"])
    steps = max(1, args.steps)
    ts = time_cpu(fn, reps=steps, warmup=max(1, args.warmup), budget_s=240.0)
    us = statistics.median(ts) / frac * 1e6
    sim_us, sim_note = reference_simulator_us(args.workload, G)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": "us", "n_gpus": world,
        "steps": len(ts), "warmup": args.warmup, "ms_per_step": round(us / 1e3, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (our arm's shapes and seeds, drawn by the host generator)",
        "config": config,
        "cpu_baseline": {"value": round(us, 1), "unit": "us", "cores": blas_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(us, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulator": {"us_per_pass": None if sim_us is None else round(sim_us, 1), "cores": 1,
                                "what": sim_note},
    }))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ficco", choices=["ficco", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--kinds", default="", help="comma-separated subset of schedules for the variants table")
    ap.add_argument("--kind", default="", help="override the headline schedule (default: the selector's choice)")
    ap.add_argument("--agent", default="", help="override the headline comm agent (default: the machine file's)")
    ap.add_argument("--headline-only", action="store_true", help="skip the all-variants table")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="N=1 only: the job size G this GPU plays rank 0 of (default 8; C1: 4; C3 is quoted at "
                         "G = 2, 4 and 8)")
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

"""Analytic executor: discrete-event pricing of an ExecutionPlan.

Mirror of the reference executor slot (/root/reference/pkg/src/overlap_sim/
engine.py:35-318): same public names (``simulate``, ``speedup``,
``base_duration``, ``SimResult``, ``TaskSpan``, ``DeadlockError``,
``export_trace_csv``) and the same arithmetic, so makespans agree with the
reference to the last bit on the golden scenarios.

On B200 the *real* executor is ``executor.execute`` (CUDA streams + copy
engines + the tcgen05 tile kernel); it reports its measured timeline in this
module's ``SimResult``/``TaskSpan`` schema so simulated and measured runs diff
directly. ``simulate`` stays as the cost model the selector is validated
against.

Model (engine.py:1-14): every task holds its resources for its lifetime —
GEMM: the GPU's compute engine; gather/scatter: its local-copy engine;
transfer: a DMA channel at the source plus the (src,dst) link on a mesh, or
the src NIC-out and dst NIC-in on a switch. DIL scales durations statically;
CIL gates rates dynamically (GEMM at 1/gemm_cil while any transfer touches
its GPU; transfer at 1/comm_cil while a GEMM or copy runs on either end).
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .domain import MachineConfig, Scenario, gemm_mt
from .pricing import LossModel, Topology, TopologyKind, comm_cil, comm_dil, gemm_cil, lookup, shard_scaled
from .routing import (ExecutionPlan, GatherSpec, GemmSpec, ScatterSpec, ScheduleKind, Task, TransferSpec,
                      task_label)


class DeadlockError(RuntimeError):
    """Some tasks can never start (unsatisfiable dependencies)."""


@dataclass(frozen=True)
class TaskSpan:
    task_id: int
    gpu: int
    kind: str
    start: float
    end: float
    contended_time: float

    @property
    def contended_fraction(self) -> float:
        dur = self.end - self.start
        return self.contended_time / dur if dur > 0 else 0.0


@dataclass(frozen=True)
class SimResult:
    scenario_name: str
    schedule: ScheduleKind
    makespan: float
    timeline: tuple[TaskSpan, ...]
    busy_time: dict[str, float]
    max_work_rel_error: float
    speedup_vs_serial: float | None = None


def base_duration(task: Task, machine: MachineConfig, topo: Topology, model: LossModel,
                  scenario: Scenario, ideal: bool = False) -> float:
    """Uncontended task time with DIL applied (engine.py:76-103)."""
    spec = task.kind
    if isinstance(spec, GemmSpec):
        t = spec.flops / machine.effective_flops
        if ideal:
            return t
        if spec.dil is not None:
            t *= lookup(model.gemm_dil_tables[spec.dil[0]], spec.dil[1])
        return t + machine.launch_overhead
    if isinstance(spec, TransferSpec):
        t = spec.bytes / (topo.link_bw if topo.kind is TopologyKind.MESH else topo.nic_bw)
        if spec.fine and not ideal:
            t *= comm_dil(model, spec.bytes)
        return t + topo.latency
    return 2.0 * spec.bytes / machine.effective_copy_bw  # one read + one write


def _claims(task: Task, topo: Topology) -> tuple:
    spec = task.kind
    if isinstance(spec, GemmSpec):
        return (("gemm", task.gpu),)
    if isinstance(spec, (GatherSpec, ScatterSpec)):
        return (("copy", task.gpu),)
    if topo.kind is TopologyKind.MESH:
        return (("dma", spec.src), ("link", spec.src, spec.dst))
    return (("dma", spec.src), ("nic_out", spec.src), ("nic_in", spec.dst))


def _capacities(n: int, machine: MachineConfig, topo: Topology) -> dict:
    cap = {}
    for gpu in range(n):
        cap[("gemm", gpu)] = 1
        cap[("copy", gpu)] = 1
        cap[("dma", gpu)] = machine.n_dma_engines
        if topo.kind is TopologyKind.SWITCH:
            cap[("nic_out", gpu)] = 1
            cap[("nic_in", gpu)] = 1
    if topo.kind is TopologyKind.MESH:
        for a in range(n):
            for b in range(n):
                if a != b:
                    cap[("link", a, b)] = 1
    return cap


class _EventLoop:
    """State of one simulation run (kept in one object instead of closures)."""

    def __init__(self, plan: ExecutionPlan, machine: MachineConfig, topo: Topology, model: LossModel, seed: int):
        sc = plan.scenario
        self.tasks = plan.tasks
        self.ideal = plan.schedule is ScheduleKind.IDEAL
        mt = gemm_mt(sc.gemm)
        self.gemm_mult = gemm_cil(model, mt, machine.comm_agent)
        self.xfer_mult = comm_cil(model, mt, machine.comm_agent)
        if plan.schedule is ScheduleKind.SHARD_OVERLAP_P2P:
            self.gemm_mult = shard_scaled(model, self.gemm_mult, "gemm")
            self.xfer_mult = shard_scaled(model, self.xfer_mult, "comm")
        rng = random.Random(f"{seed}:{sc.name}:{plan.schedule.value}") if machine.noise > 0 else None
        self.duration = []
        for t in self.tasks:
            d = base_duration(t, machine, topo, model, sc, ideal=self.ideal)
            if rng is not None:
                d *= 1.0 + rng.uniform(0.0, machine.noise)
            self.duration.append(d)
        self.cap = _capacities(sc.n_gpus, machine, topo)
        self.claims = [_claims(t, topo) for t in self.tasks]
        self.waiting_on = [len(t.deps) for t in self.tasks]
        self.children: dict[int, list[int]] = {}
        for t in self.tasks:
            for d in t.deps:
                self.children.setdefault(d, []).append(t.id)
        self.ready = sorted(t.id for t in self.tasks if not t.deps)
        self.left: dict[int, float] = {}  # running id -> remaining uncontended work
        self.rate: dict[int, float] = {}
        self.t0: dict[int, float] = {}
        self.gated: dict[int, float] = {}
        self.work: dict[int, float] = {}
        self.busy: dict[str, float] = {}
        self.spans: list[TaskSpan] = []
        self.now = 0.0

    def admit(self) -> None:
        keep = []
        for tid in self.ready:
            need = self.claims[tid]
            if all(self.cap[r] >= 1 for r in need):
                for r in need:
                    self.cap[r] -= 1
                self.left[tid] = self.duration[tid]
                self.t0[tid] = self.now
                self.gated[tid] = 0.0
                self.work[tid] = 0.0
            else:
                keep.append(tid)
        self.ready[:] = keep

    def rerate(self) -> None:
        if self.ideal:
            for tid in self.left:
                self.rate[tid] = 1.0
            return
        gemm_on, copy_on, xfer_on = set(), set(), set()
        for tid in self.left:
            spec = self.tasks[tid].kind
            if isinstance(spec, GemmSpec):
                gemm_on.add(self.tasks[tid].gpu)
            elif isinstance(spec, (GatherSpec, ScatterSpec)):
                copy_on.add(self.tasks[tid].gpu)
            else:
                xfer_on.update((spec.src, spec.dst))
        self.rate.clear()
        for tid in self.left:
            spec = self.tasks[tid].kind
            if isinstance(spec, GemmSpec):
                self.rate[tid] = 1.0 / self.gemm_mult if self.tasks[tid].gpu in xfer_on else 1.0
            elif isinstance(spec, TransferSpec):
                hot = (spec.src in gemm_on or spec.dst in gemm_on or spec.src in copy_on or spec.dst in copy_on)
                self.rate[tid] = 1.0 / self.xfer_mult if hot else 1.0
            else:
                self.rate[tid] = 1.0

    def advance(self) -> int:
        order = sorted(self.left)
        until = {tid: (self.left[tid] / self.rate[tid] if self.left[tid] > 0 else 0.0) for tid in order}
        step = min(until[tid] for tid in order)
        self.now += step
        for tid in order:
            did = step * self.rate[tid]
            self.work[tid] += did
            if step > 0 and self.rate[tid] < 1.0:
                self.gated[tid] += step
            self.left[tid] = 0.0 if until[tid] == step else max(0.0, self.left[tid] - did)
        finished = [tid for tid in order if until[tid] == step]
        for tid in finished:
            del self.left[tid]
            for r in self.claims[tid]:
                self.cap[r] += 1
                key = ":".join(map(str, r))
                self.busy[key] = self.busy.get(key, 0.0) + (self.now - self.t0[tid])
            t = self.tasks[tid]
            self.spans.append(TaskSpan(tid, t.gpu, task_label(t.kind), self.t0[tid], self.now, self.gated[tid]))
            for child in self.children.get(tid, ()):
                self.waiting_on[child] -= 1
                if self.waiting_on[child] == 0:
                    self.ready.append(child)
        self.ready.sort()
        return len(finished)


def simulate(plan: ExecutionPlan, machine: MachineConfig, topo: Topology, model: LossModel,
             seed: int = 0) -> SimResult:
    """Price ``plan`` to completion (engine.py:117-297)."""
    loop = _EventLoop(plan, machine, topo, model, seed)
    n, done = len(plan.tasks), 0
    while done < n:
        loop.admit()
        if not loop.left:
            stuck = [t.id for t in plan.tasks if loop.waiting_on[t.id] > 0][:5]
            raise DeadlockError(
                f"{n - done} task(s) can never start; blocked ids {loop.ready[:5]}, unmet-dependency ids {stuck}"
            )
        loop.rerate()
        done += loop.advance()
    err = 0.0
    for t in plan.tasks:
        base = loop.duration[t.id]
        if base > 0:
            err = max(err, abs(loop.work[t.id] - base) / base)
    spans = tuple(sorted(loop.spans, key=lambda s: s.task_id))
    return SimResult(plan.scenario.name, plan.schedule, loop.now, spans, loop.busy, err)


def speedup(result: SimResult, serial_result: SimResult) -> float:
    """serial makespan / this makespan."""
    if result.scenario_name != serial_result.scenario_name:
        raise ValueError(
            f"speedup compares results for different scenarios: "
            f"{result.scenario_name!r} vs {serial_result.scenario_name!r}"
        )
    return serial_result.makespan / result.makespan


def export_trace_csv(result: SimResult) -> str:
    """task_id,gpu,kind,start_s,end_s,contended_fraction (engine.py:310-318)."""
    rows = ["task_id,gpu,kind,start_s,end_s,contended_fraction"]
    rows += [f"{s.task_id},{s.gpu},{s.kind},{s.start:.9e},{s.end:.9e},{s.contended_fraction:.6f}"
             for s in result.timeline]
    return "\n".join(rows) + "\n"

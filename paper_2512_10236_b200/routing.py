"""Schedule planning: scenario -> per-GPU task DAG with exact chunk routing.

Host-side mirror of the reference planner
(/root/reference/pkg/src/overlap_sim/planner.py:34-533). Public names,
argument meaning, emitted task order (hence task ids), dependency sets and
``PlanError`` behaviour are identical so plans compare field-for-field with
the reference (pinned by ``tests/golden/plans_*.json``).

Notation: G ranks, R = M/G rows per shard, r = M/G^2 rows per
fine chunk, b = K/G columns per 2D block, e = element bytes.

The routing every fine-grain schedule shares (planner.py:152-167): G
all-to-all rounds; in round c GPU ``src`` sends its fine chunk c, i.e. rows
``[src*R + c*r, +r)`` of the gathered operand, to every other GPU. On B200 the
executor lowers each transfer to a copy-engine copy landing directly at that
row offset of the destination's gathered buffer, so the reference's
``GatherSpec``/``ScatterSpec`` bookkeeping tasks become no-ops
(see ``lowering.py``).
"""

from __future__ import annotations

import csv
import enum
import io
from dataclasses import dataclass

from .domain import GemmShape, Scenario, gemm_flops, gemm_otb
from .pricing import Topology


class PlanError(ValueError):
    """The scenario cannot be expanded into the requested schedule."""


class ScheduleKind(enum.Enum):
    SERIAL = "serial"
    IDEAL = "ideal"
    SHARD_OVERLAP_P2P = "shard_overlap_p2p"
    UNIFORM_FUSED_1D = "uniform_fused_1d"
    HETERO_FUSED_1D = "hetero_fused_1d"
    HETERO_UNFUSED_1D = "hetero_unfused_1d"
    UNIFORM_FUSED_2D = "uniform_fused_2d"


# Enum order doubles as the tie-break order of the exhaustive search.
FINE_GRAIN_KINDS = tuple(ScheduleKind)[3:]
ALL_KINDS = tuple(ScheduleKind)


@dataclass(frozen=True)
class TransferSpec:
    src: int
    dst: int
    bytes: int
    fine: bool  # fine-grain chunk (pays comm DIL) vs full shard
    round_idx: int = 0


@dataclass(frozen=True)
class GatherSpec:
    bytes: int


@dataclass(frozen=True)
class ScatterSpec:
    bytes: int


@dataclass(frozen=True)
class GemmSpec:
    shape: GemmShape
    additive: bool = False
    dil: tuple[str, float] | None = None  # (loss table key, lookup x)
    rows: tuple[tuple[int, int], ...] = ()  # output row fragments (start, count)
    col_block: tuple[int, int] | None = None  # K block (start, count) for 2D

    @property
    def flops(self) -> int:
        return gemm_flops(self.shape)


TaskSpec = TransferSpec | GatherSpec | ScatterSpec | GemmSpec


@dataclass(frozen=True)
class Task:
    id: int
    gpu: int  # executing GPU; for transfers the destination
    kind: TaskSpec
    deps: tuple[int, ...] = ()


@dataclass(frozen=True)
class ExecutionPlan:
    schedule: ScheduleKind
    scenario: Scenario
    tasks: tuple[Task, ...]
    chunk_rows: int | None = None
    chunk_cols: int | None = None

    @property
    def n_gpus(self) -> int:
        return self.scenario.n_gpus


class _Dag:
    """Append-only task list; ids are emission indices (topological order)."""

    def __init__(self) -> None:
        self.tasks: list[Task] = []

    def emit(self, gpu: int, spec: TaskSpec, deps=()) -> int:
        tid = len(self.tasks)
        self.tasks.append(Task(tid, gpu, spec, tuple(deps)))
        return tid


@dataclass(frozen=True)
class _Geometry:
    """Chunk geometry of one scenario (all integers)."""

    g: int
    shape: GemmShape

    @property
    def shard_rows(self) -> int:  # R
        return self.shape.m // self.g

    @property
    def chunk_rows(self) -> int:  # r
        return self.shape.m // (self.g * self.g)

    @property
    def shard_bytes(self) -> int:
        return self.shard_rows * self.shape.k * self.shape.elt_bytes

    @property
    def chunk_bytes(self) -> int:
        s = self.shape
        return s.m * s.k * s.elt_bytes // (self.g * self.g)

    def rows_shape(self, m: int) -> GemmShape:
        s = self.shape
        return GemmShape(m=m, n=s.n, k=s.k, elt_bytes=s.elt_bytes)

    def chunk_start(self, owner: int, c: int) -> int:
        """First gathered row of fine chunk c of ``owner``'s shard."""
        return owner * self.shard_rows + c * self.chunk_rows


def _divisible(scenario: Scenario, label: str, value: int, degree: int) -> None:
    if value % degree:
        raise PlanError(f"scenario {scenario.name!r}: {label}={value} is not divisible by {degree}")


def _topo_matches(scenario: Scenario, topo: Topology | None) -> None:
    if topo is not None and topo.n_gpus != scenario.n_gpus:
        raise PlanError(
            f"topology has {topo.n_gpus} GPUs but scenario {scenario.name!r} "
            f"expects {scenario.n_gpus}"
        )


def _fine_geometry(scenario: Scenario) -> _Geometry:
    g = scenario.n_gpus
    _divisible(scenario, "M", scenario.gemm.m, g * g)
    return _Geometry(g, scenario.gemm)


def _a2a(dag: _Dag, g: int, nbytes: int) -> list[list[list[int]]]:
    """G all-to-all rounds; returns arrivals[dst][round] = transfer ids (src ascending).

    planner.py:152-167. No explicit dependencies: rounds are ordered by
    per-link exclusivity and ascending ids.
    """
    arrivals = [[[] for _ in range(g)] for _ in range(g)]
    for rnd in range(g):
        for dst in range(g):
            for src in range(g):
                if src != dst:
                    arrivals[dst][rnd].append(
                        dag.emit(dst, TransferSpec(src=src, dst=dst, bytes=nbytes, fine=True, round_idx=rnd))
                    )
    return arrivals


def plan_serial(scenario: Scenario, topo: Topology | None = None) -> ExecutionPlan:
    """No-overlap baseline: whole-shard all-gather, then one full GEMM (planner.py:170-191)."""
    _topo_matches(scenario, topo)
    g = scenario.n_gpus
    _divisible(scenario, "M", scenario.gemm.m, g)
    geo = _Geometry(g, scenario.gemm)
    dag = _Dag()
    for dst in range(g):
        xfers = [dag.emit(dst, TransferSpec(src=s, dst=dst, bytes=geo.shard_bytes, fine=False))
                 for s in range(g) if s != dst]
        dag.emit(dst, GemmSpec(shape=scenario.gemm, rows=((0, scenario.gemm.m),)), deps=xfers)
    return ExecutionPlan(ScheduleKind.SERIAL, scenario, tuple(dag.tasks))


def plan_shard_overlap(scenario: Scenario, topo: Topology | None = None) -> ExecutionPlan:
    """Shard-granularity P2P ring (planner.py:194-240).

    Step i on GPU g multiplies shard (g - i) mod G; the step-i shard arrives
    from the left neighbour (g-1) mod G, store-and-forward from step 2 on.
    """
    _topo_matches(scenario, topo)
    g = scenario.n_gpus
    _divisible(scenario, "M", scenario.gemm.m, g)
    geo = _Geometry(g, scenario.gemm)
    step_shape = geo.rows_shape(geo.shard_rows)
    dil = ("row8", gemm_otb(scenario.gemm))
    dag = _Dag()

    def gemm(gpu: int, step: int, deps=()) -> int:
        owner = (gpu - step) % g
        rows = ((owner * geo.shard_rows, geo.shard_rows),)
        return dag.emit(gpu, GemmSpec(shape=step_shape, dil=dil, rows=rows), deps)

    last_gemm = [gemm(gpu, 0) for gpu in range(g)]
    last_xfer: list[int] | None = None
    for step in range(1, g):
        xfer = []
        for gpu in range(g):
            left = (gpu - 1) % g
            deps = [last_xfer[left]] if last_xfer is not None else []
            xfer.append(dag.emit(gpu, TransferSpec(src=left, dst=gpu, bytes=geo.shard_bytes,
                                                   fine=False, round_idx=step - 1), deps))
        last_gemm = [gemm(gpu, step, (last_gemm[gpu], xfer[gpu])) for gpu in range(g)]
        last_xfer = xfer
    return ExecutionPlan(ScheduleKind.SHARD_OVERLAP_P2P, scenario, tuple(dag.tasks))


def _uniform_steps(scenario: Scenario, copies: bool) -> ExecutionPlan:
    """uniform_fused_1d (copies=True) and ideal (copies=False): planner.py:249-273.

    Step s on every GPU multiplies fine chunk s of every shard (local one
    included): rows ``{p*R + s*r : p}``.
    """
    geo = _fine_geometry(scenario)
    g, s_ = geo.g, scenario.gemm
    step_shape = geo.rows_shape(geo.shard_rows)
    dil = ("row8", gemm_otb(s_)) if copies else None
    dag = _Dag()
    arrivals = _a2a(dag, g, geo.chunk_bytes)
    for step in range(g):
        rows = tuple((geo.chunk_start(p, step), geo.chunk_rows) for p in range(g))
        for gpu in range(g):
            deps = arrivals[gpu][step]
            if copies:
                deps = [dag.emit(gpu, GatherSpec(bytes=geo.shard_rows * s_.k * s_.elt_bytes), deps)]
            gid = dag.emit(gpu, GemmSpec(shape=step_shape, dil=dil, rows=rows), deps)
            if copies:
                dag.emit(gpu, ScatterSpec(bytes=geo.shard_rows * s_.n * s_.elt_bytes), [gid])
    kind = ScheduleKind.UNIFORM_FUSED_1D if copies else ScheduleKind.IDEAL
    return ExecutionPlan(kind, scenario, tuple(dag.tasks), chunk_rows=geo.chunk_rows)


def plan_ideal(scenario: Scenario, topo: Topology | None = None) -> ExecutionPlan:
    """Loss-free pipelining bound: same DAG as uniform_fused_1d minus copies and DIL."""
    _topo_matches(scenario, topo)
    return _uniform_steps(scenario, copies=False)


def _hetero(scenario: Scenario, fused: bool) -> ExecutionPlan:
    """Local shard first, then remote chunks (planner.py:291-348).

    fused: one GEMM per round over the G-1 remote chunks (DIL ``row8`` at the
    fused shape's own OTB). unfused: one GEMM per (round, peer), each gated by
    exactly its own transfer (DIL ``row64`` at the parent OTB).
    """
    geo = _fine_geometry(scenario)
    g, parent = geo.g, scenario.gemm
    dag = _Dag()
    for gpu in range(g):
        dag.emit(gpu, GemmSpec(shape=geo.rows_shape(geo.shard_rows), dil=("row8", gemm_otb(parent)),
                               rows=((gpu * geo.shard_rows, geo.shard_rows),)))
    arrivals = _a2a(dag, g, geo.chunk_bytes)
    if fused:
        shape = geo.rows_shape((g - 1) * geo.chunk_rows)
        dil = ("row8", gemm_otb(shape))
        for step in range(g):
            for gpu in range(g):
                rows = tuple((geo.chunk_start(p, step), geo.chunk_rows) for p in range(g) if p != gpu)
                dag.emit(gpu, GemmSpec(shape=shape, dil=dil, rows=rows), arrivals[gpu][step])
        kind = ScheduleKind.HETERO_FUSED_1D
    else:
        shape = geo.rows_shape(geo.chunk_rows)
        dil = ("row64", gemm_otb(parent))
        for step in range(g):
            for gpu in range(g):
                peers = [p for p in range(g) if p != gpu]
                for xfer_id, p in zip(arrivals[gpu][step], peers):
                    dag.emit(gpu, GemmSpec(shape=shape, dil=dil, rows=((geo.chunk_start(p, step), geo.chunk_rows),)),
                             [xfer_id])
        kind = ScheduleKind.HETERO_UNFUSED_1D
    return ExecutionPlan(kind, scenario, tuple(dag.tasks), chunk_rows=geo.chunk_rows)


def _column_blocks(scenario: Scenario) -> ExecutionPlan:
    """uniform_fused_2d (planner.py:351-390).

    Round c ships the R x b slab ``A[src*R:+R, c*b:+b]`` to every peer; step s
    is an additive (M, N, b) GEMM over K-block s, chained on step s-1.
    """
    g, s_ = scenario.n_gpus, scenario.gemm
    _divisible(scenario, "M", s_.m, g)
    _divisible(scenario, "K", s_.k, g)
    big_r, b = s_.m // g, s_.k // g
    step_shape = GemmShape(m=s_.m, n=s_.n, k=b, elt_bytes=s_.elt_bytes)
    dil = ("col8", gemm_otb(step_shape))
    dag = _Dag()
    arrivals = _a2a(dag, g, big_r * b * s_.elt_bytes)
    prev: list[int | None] = [None] * g
    for step in range(g):
        for gpu in range(g):
            gather = dag.emit(gpu, GatherSpec(bytes=s_.m * b * s_.elt_bytes), arrivals[gpu][step])
            deps = [gather] if prev[gpu] is None else [gather, prev[gpu]]
            prev[gpu] = dag.emit(gpu, GemmSpec(shape=step_shape, additive=True, dil=dil,
                                               rows=((0, s_.m),), col_block=(step * b, b)), deps)
    return ExecutionPlan(ScheduleKind.UNIFORM_FUSED_2D, scenario, tuple(dag.tasks),
                         chunk_rows=big_r, chunk_cols=b)


_FINE_PLANNERS = {
    ScheduleKind.UNIFORM_FUSED_1D: lambda s: _uniform_steps(s, copies=True),
    ScheduleKind.HETERO_FUSED_1D: lambda s: _hetero(s, fused=True),
    ScheduleKind.HETERO_UNFUSED_1D: lambda s: _hetero(s, fused=False),
    ScheduleKind.UNIFORM_FUSED_2D: _column_blocks,
}


def plan_fine_overlap(scenario: Scenario, topo: Topology | None = None,
                      kind: ScheduleKind = ScheduleKind.UNIFORM_FUSED_1D) -> ExecutionPlan:
    """Expand one of the four fine-grain schedules."""
    _topo_matches(scenario, topo)
    planner = _FINE_PLANNERS.get(kind)
    if planner is None:
        raise PlanError(f"{kind} is not a fine-grain overlap schedule")
    return planner(scenario)


def build_plan(scenario: Scenario, kind: ScheduleKind, topo: Topology | None = None) -> ExecutionPlan:
    """Plan any schedule kind (planner.py:409-417)."""
    if kind is ScheduleKind.SERIAL:
        return plan_serial(scenario, topo)
    if kind is ScheduleKind.IDEAL:
        return plan_ideal(scenario, topo)
    if kind is ScheduleKind.SHARD_OVERLAP_P2P:
        return plan_shard_overlap(scenario, topo)
    return plan_fine_overlap(scenario, topo, kind)


def supported_kinds(scenario: Scenario) -> list[ScheduleKind]:
    """Fine-grain kinds whose divisibility constraints hold (planner.py:420-429)."""
    ok = []
    for kind in FINE_GRAIN_KINDS:
        try:
            build_plan(scenario, kind)
        except PlanError:
            continue
        ok.append(kind)
    return ok


def _coverage(spans, total: int, gpu: int, what: str, dim: str) -> list[str]:
    at = 0
    for start, count in sorted(spans):
        if start != at:
            return [f"gpu {gpu}: {what} coverage gap/overlap at {start}"]
        at = start + count
    if at != total:
        return [f"gpu {gpu}: {what} coverage ends at {at} != {dim}={total}"]
    return []


def validate_plan(plan: ExecutionPlan, scenario: Scenario | None = None) -> list[str]:
    """Conservation (ingress, flops), exact coverage and DAG sanity (planner.py:438-514)."""
    scenario = scenario or plan.scenario
    g, s_ = scenario.n_gpus, scenario.gemm
    problems: list[str] = []
    ingress, flops = [0] * g, [0] * g
    for t in plan.tasks:
        spec = t.kind
        if isinstance(spec, TransferSpec):
            if spec.src == spec.dst:
                problems.append(f"task {t.id}: transfer src == dst == {spec.src}")
            if spec.bytes <= 0:
                problems.append(f"task {t.id}: transfer bytes must be positive")
            ingress[spec.dst] += spec.bytes
        elif isinstance(spec, GemmSpec):
            flops[t.gpu] += spec.flops
        elif spec.bytes <= 0:
            problems.append(f"task {t.id}: copy bytes must be positive")
    want_in = (g - 1) * (s_.m // g) * s_.k * s_.elt_bytes
    problems += [f"gpu {i}: ingress bytes {v} != expected {want_in}" for i, v in enumerate(ingress) if v != want_in]
    want_f = 2 * s_.m * s_.n * s_.k
    problems += [f"gpu {i}: gemm flops {v} != expected {want_f}" for i, v in enumerate(flops) if v != want_f]
    gemms = [t for t in plan.tasks if isinstance(t.kind, GemmSpec)]
    for gpu in range(g):
        if plan.schedule is ScheduleKind.UNIFORM_FUSED_2D:
            spans = [t.kind.col_block for t in gemms if t.gpu == gpu and t.kind.col_block]
            problems += _coverage(spans, s_.k, gpu, "column", "K")
        else:
            spans = [f for t in gemms if t.gpu == gpu for f in t.kind.rows]
            problems += _coverage(spans, s_.m, gpu, "row", "M")
    ids = {t.id for t in plan.tasks}
    for t in plan.tasks:
        for d in t.deps:
            if d not in ids:
                problems.append(f"task {t.id}: unknown dep {d}")
            elif d >= t.id:
                problems.append(f"task {t.id}: dep {d} is not topologically earlier")
    return problems


def task_label(spec: TaskSpec) -> str:
    if isinstance(spec, TransferSpec):
        return f"transfer[{spec.src}->{spec.dst}]"
    if isinstance(spec, GatherSpec):
        return "gather"
    if isinstance(spec, ScatterSpec):
        return "scatter"
    return "gemm"


def export_plan_csv(plan: ExecutionPlan) -> str:
    """task_id,gpu,kind,bytes,flops,deps (planner.py:517-533)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["task_id", "gpu", "kind", "bytes", "flops", "deps"])
    for t in plan.tasks:
        spec = t.kind
        nbytes = 0 if isinstance(spec, GemmSpec) else spec.bytes
        nflops = spec.flops if isinstance(spec, GemmSpec) else 0
        w.writerow([t.id, t.gpu, task_label(spec), nbytes, nflops, " ".join(map(str, t.deps))])
    return buf.getvalue()

"""Overlapped-op entry points (the north star's additions to the reference API).

* ``all_gather_matmul(a_shard, weight)``        AG -> GEMM      (TP/SP up-projection, configs C1/C2/C3')
* ``matmul_reduce_scatter(a, weight)``          GEMM -> RS      (TP/SP down-projection, config C3)
* ``cp_kv_all_gather_qk(q, k_shard)``           CP KV-AG -> QK^T (config C4)

Each builds the reference's ExecutionPlan for the equivalent scenario
(``routing.build_plan``), picks the schedule with ``select_schedule`` when
``kind`` is None, lowers it for this rank (``lowering``) and runs it through
the C-ABI executor. Weights use the ``nn.Linear`` layout ``[N, K]`` (K
contiguous), so C = A @ W^T.

A ``FiccoGroup`` owns the communicator (symmetric workspaces, copy stream,
epoch) and caches lowered plans per (op, shape, kind). Two flavours:

* ``FiccoGroup.distributed(group)`` — one process per GPU (or several ranks
  sharing a GPU), CUDA-IPC handles exchanged through ``torch.distributed``.
* ``FiccoGroup.virtual_group(world, rank)`` — decomposition-only single-process
  mode: this process plays ``rank`` of a ``world``-rank job whose peers'
  shards are pre-loaded into local stand-in workspaces (``load_peer_shards``)
  so the copy engines, flags and tile kernel do exactly one rank's work.
"""

from __future__ import annotations

import math
import os

import torch

from .domain import Collective, GemmShape, Parallelism, Scenario
from .lowering import Lowered, lower_ag, lower_rs
from .machines import b200_machine
from .routing import PlanError, ScheduleKind, build_plan
from .runtime import FICCO_WS_DATA_OFFSET, Communicator, Plan
from .selector import select_schedule


# FICCO_SERIALIZE=1: run copy programs to completion before the tile kernel (kernel
# profilers such as ncu serialise work, which would starve flag-gated tiles). ncu is
# detected by the environment it injects (NV_COMPUTE_PROFILER_PERFWORKS_DIR) and switches this on by itself.
SERIALIZE = os.environ.get("FICCO_SERIALIZE", "0") == "1" or bool(os.environ.get("NV_COMPUTE_PROFILER_PERFWORKS_DIR"))


def _scenario(name: str, m: int, n: int, k: int, world: int, collective=Collective.ALL_GATHER) -> Scenario:
    par = Parallelism.EP if collective is Collective.ALL_TO_ALL else Parallelism.SP_TP
    return Scenario(name=name, parallelism=par, model="ficco-op", gemm=GemmShape(m, n, k, 2),
                    collective=collective, n_gpus=world)


def choose_kind(scenario: Scenario, kind: ScheduleKind | str | None, machine=None, t_ref: float | None = None):
    if kind is None:
        spec = machine or b200_machine()
        return select_schedule(scenario, spec.machine, spec.t_ref if t_ref is None else t_ref)
    return ScheduleKind(kind) if isinstance(kind, str) else kind


class FiccoGroup:
    def __init__(self, world: int, rank: int, virtual: bool, pg=None):
        self.world, self.rank, self.virtual, self.pg = world, rank, virtual, pg
        self.comm: Communicator | None = None
        self._plans: dict = {}
        self._fast: dict = {}
        self._ws_bytes = 0
        self.device: int | None = None  # CUDA device of the workspaces (set with the first workspace)
        self._mc = None                  # runtime.Multicast: the NVLS workspace (comm_agent = nvls), lazily
        self._ws_views: dict = {}        # rank -> uint8 view of its whole workspace (this communicator's)

    @classmethod
    def virtual_group(cls, world: int, rank: int = 0) -> "FiccoGroup":
        return cls(world, rank, True)

    @classmethod
    def distributed(cls, group=None) -> "FiccoGroup":
        import torch.distributed as dist
        return cls(dist.get_world_size(group), dist.get_rank(group), False, group)

    # ---------------------------------------------------------------- workspace
    def ensure_workspace(self, nbytes: int) -> None:
        nbytes = max(nbytes, FICCO_WS_DATA_OFFSET)
        if self.comm is not None and nbytes <= self._ws_bytes:
            return
        nbytes = 1 << max(20, math.ceil(math.log2(nbytes)))
        self._retire()
        if self.virtual:
            self.comm = Communicator.virtual(self.world, self.rank, nbytes)
        else:
            self.comm = Communicator.from_process_group(nbytes, self.pg)
        self._ws_bytes = nbytes
        self.device = torch.cuda.current_device()
        if self._mc is not None:
            self.comm.set_multicast(self._mc)

    def ensure_multicast(self, nbytes: int) -> None:
        """The group's NVLS multicast workspace of at least `nbytes` (collective in a distributed group;
        raises NotImplementedError where the fabric gives no multicast objects)."""
        if self.virtual:
            raise PlanError("comm_agent='nvls' needs real ranks on distinct GPUs; virtual peers share one device")
        if self._mc is not None and self._mc.nbytes >= nbytes:
            return
        from .runtime import Multicast
        torch.cuda.synchronize()
        self._barrier()
        if self._mc is not None:
            for plan, _ in self._plans.values():
                plan.close()
            self._plans.clear()
            self._fast.clear()
            self._mc.release()
            self._mc = None
        self._mc = Multicast(nbytes, self.pg)
        if self.comm is not None:
            self.comm.set_multicast(self._mc)

    def _barrier(self) -> None:
        if not self.virtual:
            import torch.distributed as dist
            dist.barrier(group=self.pg)

    def _retire(self) -> None:
        """Free the plans and the communicator without pulling memory from under a peer.

        A peer may still be pulling from our workspace, notifying into our flag block or
        TMA-storing into our receive slots when we finish our last call, so in a distributed
        group every rank first drains its own work (synchronize) and meets the others
        (barrier): after that no rank has device work touching any workspace. Each rank then
        unmaps the peers' workspaces, meets them again, and only then frees its own — the
        IPC mappings of it in other processes are gone by then (CUDA leaves freeing memory
        that peers still map undefined).
        """
        if self.comm is None:
            return
        self._ws_views.clear()
        torch.cuda.synchronize()
        self._barrier()
        for plan, _ in self._plans.values():
            plan.close()
        self._plans.clear()
        self._fast.clear()
        self.comm.close(between=self._barrier)
        self.comm = None

    def plan(self, key, make) -> tuple[Plan, Lowered]:
        hit = self._plans.get(key)
        if hit is None:
            low = make()
            self.ensure_workspace(low.ws_bytes)
            if low.mc_bytes:
                self.ensure_multicast(low.mc_bytes)
            hit = (Plan(self.comm, low.desc, low.ops, low.tiles), low)
            self._plans[key] = hit
        return hit

    def ws_tensor(self, rank: int, offset: int, shape, dtype=torch.bfloat16) -> torch.Tensor:
        """A torch view of (part of) a workspace (local, or a virtual peer's).

        Views are slices of one byte tensor per workspace, wrapped once per communicator: wrapping a raw
        pointer costs ~40 us of host time, slicing a few (input_slot / kv_slot run before every call)."""
        nbytes = math.prod(shape) * dtype.itemsize
        if offset + nbytes > self._ws_bytes:
            raise ValueError("view exceeds workspace")
        whole = self._ws_views.get(rank)
        if whole is None:
            whole = _wrap_device_ptr(self.comm.ws_ptrs[rank], (self._ws_bytes,), torch.uint8)
            self._ws_views[rank] = whole
        return whole[offset:offset + nbytes].view(dtype).view(*shape)

    def input_slot(self, rows: int, cols: int, n_out: int, kind=None) -> torch.Tensor:
        """This rank's slot of the gathered buffer for the NEXT all_gather_matmul call.

        Writing the shard here (e.g. as the producing layer's output) and passing
        the view as ``a_shard`` skips the local publish copy: peers pull it
        straight from the slot. The slot alternates between calls (workspace
        parity), so ask for it before every call.
        """
        _, low, _ = prepare_ag(self, rows, cols, n_out, kind)
        par = self.comm.epoch() & 1
        off = low.gather_off + par * low.gather_par + self.rank * rows * cols * 2
        return self.ws_tensor(self.rank, off, (rows, cols))

    def kv_slot(self, tq: int, d: int, tkv: int, kind=None, scale: float | None = None) -> torch.Tensor:
        """This rank's K-shard slot [tkv / world, d] of the gathered K for the NEXT cp_kv_all_gather_qk call
        (the context-parallel twin of ``input_slot``: write the shard here and pass the view as ``k_shard``)."""
        _, low, _ = prepare_cp(self, tq, d, tkv, kind, scale)
        rows = tkv // self.world
        par = self.comm.epoch() & 1
        off = low.gather_off + par * low.gather_par + self.rank * rows * d * 2
        return self.ws_tensor(self.rank, off, (rows, d))

    def close(self) -> None:
        """Release the group (collective for distributed groups: every rank must call it)."""
        self._retire()
        if self._mc is not None:
            self._barrier()
            self._mc.release()
            self._mc = None

    # ---------------------------------------------------------------- virtual-mode data
    def load_peer_shards(self, low: Lowered, shards: list[torch.Tensor]) -> None:
        """Virtual mode: give every stand-in peer the shards it would hold (all slots, both parities).

        Pull copies read chunk (p, c) from peer p's own slot (fine-grain kinds)
        or a forwarded shard from the left neighbour's slot (ring), so each
        peer workspace gets every shard at its gathered-row offset.
        """
        assert self.virtual
        rows = shards[0].shape[0]
        cols = shards[0].shape[1]
        for peer in range(self.world):
            if peer == self.rank:
                continue
            for p, sh in enumerate(shards):
                for par in (0, 1):
                    off = low.gather_off + par * low.gather_par + p * rows * cols * 2
                    self.ws_tensor(peer, off, (rows, cols)).copy_(sh)

    def load_peer_sends(self, low: Lowered, blocks: list[torch.Tensor]) -> None:
        """Virtual mode (all-to-all): ``blocks[p]`` = peer p's [R, K] block addressed to this rank,
        placed in p's send area (both parities) where this rank's pulls read it."""
        assert self.virtual
        rows, cols = blocks[0].shape
        for p, blk in enumerate(blocks):
            if p == self.rank:
                continue
            for par in (0, 1):
                off = low.send_off + par * low.send_par + self.rank * rows * cols * 2
                self.ws_tensor(p, off, (rows, cols)).copy_(blk)

    def load_peer_partials(self, low: Lowered, partials: list[torch.Tensor]) -> None:
        """Virtual mode (RS): ``partials[j]`` = peer slot j's [R, N] contribution to this rank's shard."""
        assert self.virtual
        rows, cols = partials[0].shape
        for j, part in enumerate(partials):
            for par in (0, 1):
                off = low.recv_off + par * low.recv_par + j * low.recv_slot
                self.ws_tensor(self.rank, off, (rows, cols)).copy_(part)
                if not low.recv_par:
                    break


def _wrap_device_ptr(ptr: int, shape, dtype) -> torch.Tensor:
    class _Holder:
        pass

    h = _Holder()
    nbytes = math.prod(shape) * dtype.itemsize
    h.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                  "strides": None}
    raw = torch.as_tensor(h, device=torch.device("cuda", torch.cuda.current_device()))
    return raw.view(dtype).view(*shape)


def _default_group(group, world):
    if group is not None:
        return group
    raise ValueError("pass a FiccoGroup (FiccoGroup.distributed(pg) or FiccoGroup.virtual_group(world, rank))")


def _check_tensor(name: str, t, shape=None, device=None) -> None:
    """Validate a call argument before its pointer crosses the C-ABI (the library sizes its TMA maps
    and copies from the plan, so a wrong dtype, stride, shape or device would read or write out of
    bounds instead of failing). Raises ValueError, like the reference API's invariant checks."""
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if t.dtype != torch.bfloat16:
        raise ValueError(f"{name} must be bfloat16 (the B200 executor computes bf16 x bf16 -> fp32), got {t.dtype}")
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor, got device {t.device}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (row-major, unit column stride)")
    if t.data_ptr() % 16:
        raise ValueError(f"{name} must be 16-byte aligned (TMA / copy-engine rows)")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _check_call(grp: FiccoGroup, args: dict, out, out_shape) -> torch.device:
    """All operands on the group's device, bf16, contiguous; ``out`` (if given) of ``out_shape``."""
    dev = None
    for name, (t, shape) in args.items():
        _check_tensor(name, t, shape, dev)
        dev = t.device
    if dev.index != torch.cuda.current_device():
        raise ValueError(f"operands are on {dev}, but the current CUDA device is cuda:{torch.cuda.current_device()}"
                         " (the group's workspaces and streams live there)")
    if grp.device is not None and dev.index != grp.device:
        raise ValueError(f"operands are on {dev}, but this FiccoGroup runs on cuda:{grp.device}")
    if out is not None:
        _check_tensor("out", out, out_shape, dev)
    return dev


def _cached(grp: FiccoGroup, key, make):
    """Per-call fast path: (plan, lowered, kind) memoised per (op, shape, requested kind)."""
    hit = grp._fast.get(key)
    if hit is None or hit[0].handle is None:
        hit = make()
        grp._fast[key] = hit
    return hit


def prepare_ag(grp: FiccoGroup, R: int, K: int, N: int, kind=None, inplace: bool = False, comm_agent=None):
    """Build (or fetch) the lowered AG->GEMM plan for this rank: (plan, lowered, kind)."""
    comm_agent = _agent(comm_agent, "ag")
    def make():
        M = R * grp.world
        sc = _scenario("ag_gemm", M, N, K, grp.world)
        kd = choose_kind(sc, kind)
        plan, low = grp.plan(("ag", M, N, K, kd, inplace, comm_agent),
                             lambda: lower_ag(build_plan(sc, kd), grp.rank, "A", inplace=inplace,
                                              comm_agent=comm_agent))
        return plan, low, kd
    return _cached(grp, ("ag", R, K, N, kind, inplace, comm_agent), make)


def prepare_a2a(grp: FiccoGroup, R: int, K: int, N: int, kind=None, comm_agent=None):
    """All-to-all (EP dispatch) -> expert GEMM plan for this rank: (plan, lowered, kind)."""
    comm_agent = _agent(comm_agent, "a2a")
    def make():
        M = R * grp.world
        sc = _scenario("a2a_gemm", M, N, K, grp.world, Collective.ALL_TO_ALL)
        kd = choose_kind(sc, kind)
        plan, low = grp.plan(("a2a", M, N, K, kd, comm_agent),
                             lambda: lower_ag(build_plan(sc, kd), grp.rank, "A", comm_agent=comm_agent))
        return plan, low, kd
    return _cached(grp, ("a2a", R, K, N, kind, comm_agent), make)


def _is_slot(grp: FiccoGroup, t: torch.Tensor, low) -> bool:
    """Is ``t`` this rank's slot of the gathered buffer for the next call's parity?"""
    if grp.comm is None or not t.is_contiguous():
        return False
    par = grp.comm.epoch() & 1
    rows, cols = t.shape
    want = grp.comm.local_ws + low.gather_off + par * low.gather_par + grp.rank * rows * cols * 2
    return t.data_ptr() == want


def prepare_rs(grp: FiccoGroup, M: int, K: int, N: int, kind=None, comm_agent=None):
    comm_agent = _agent(comm_agent, "rs")
    def make():
        sc = _scenario("gemm_rs", M, N, K, grp.world)
        kd = choose_kind(sc, kind)
        plan, low = grp.plan(("rs", M, N, K, kd, comm_agent),
                             lambda: lower_rs(sc, kd, grp.rank, virtual=grp.virtual, comm_agent=comm_agent))
        return plan, low, kd
    return _cached(grp, ("rs", M, K, N, kind, comm_agent), make)


def prepare_cp(grp: FiccoGroup, Tq: int, d: int, Tkv: int, kind=None, scale: float | None = None,
               comm_agent=None, inplace: bool = False):
    comm_agent = _agent(comm_agent, "cp")
    def make():
        sc = _scenario("cp_qk", Tkv, Tq, d, grp.world)
        kd = choose_kind(sc, kind)
        alpha = (1.0 / math.sqrt(d)) if scale is None else scale
        plan, low = grp.plan(("cp", Tkv, Tq, d, kd, alpha, inplace, comm_agent),
                             lambda: lower_ag(build_plan(sc, kd), grp.rank, "B", alpha=alpha, other_rows=Tq,
                                              inplace=inplace, comm_agent=comm_agent))
        return plan, low, kd
    return _cached(grp, ("cp", Tq, d, Tkv, kind, scale, inplace, comm_agent), make)


def default_agent(op: str) -> str:
    """The comm agent an op uses when the caller passes comm_agent=None.

    All-gather-shaped ops (AG -> GEMM, CP KV-AG -> QK^T, EP all-to-all -> GEMM) use the B200 machine file's
    agent (the reference's MachineConfig.comm_agent, machines.py:48): 'dma', copy-engine transfers, the
    north star's DMA offload. GEMM -> reduce-scatter uses 'core': on this executor that is the fused
    GEMM + RS kernel (remote tiles' epilogues TMA-store their partials straight into the owners' receive
    slots over peer memory; no partial buffer, no copy-engine round trip), which measured faster than
    copy-engine pushes on every RS shape (C3 at G = 2, 4, 8).
    """
    if op == "rs":
        return "core"
    return b200_machine().machine.comm_agent.value


def _agent(comm_agent, op: str = "ag") -> str:
    if comm_agent is None:
        return default_agent(op)
    return getattr(comm_agent, "value", comm_agent)


def _run(grp: FiccoGroup, plan: Plan, op: str, a, b, c, stream) -> None:
    if SERIALIZE:
        plan.run_parts(a, b, c, stream, tiles=2)
    else:
        plan.run_op(op, a, b, c, stream)


def all_gather_matmul(a_shard: torch.Tensor, weight: torch.Tensor, kind=None, group: FiccoGroup | None = None,
                      out: torch.Tensor | None = None, stream=None, return_gathered: bool = False,
                      comm_agent: str | None = None):
    """C = all_gather(A_shard) @ W^T with FiCCO overlap. A_shard [R, K], W [N, K] -> C [G*R, N].

    ``return_gathered`` also returns the gathered A (a view into the group's
    double-buffered workspace, valid until the call after next). ``comm_agent``
    'dma' moves chunks with the copy engines, 'core' with SM copy kernels (None:
    the B200 machine file's agent).
    """
    grp = _default_group(group, None)
    _check_tensor("a_shard", a_shard)
    R, K = a_shard.shape
    _check_tensor("weight", weight)
    N = weight.shape[0]
    M = R * grp.world
    _check_call(grp, {"a_shard": (a_shard, None), "weight": (weight, (N, K))}, out, (M, N))
    agent = _agent(comm_agent)
    plan, low, kd = prepare_ag(grp, R, K, N, kind, comm_agent=agent)
    if _is_slot(grp, a_shard, low):  # zero-copy publish: the shard already sits in its slot
        plan, low, _ = prepare_ag(grp, R, K, N, kd, inplace=True, comm_agent=agent)
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a_shard.device)
    _run(grp, plan, "ag_gemm", a_shard, weight, out, stream)
    if return_gathered:
        par = (grp.comm.epoch() - 1) & 1  # parity of the run just enqueued
        gathered = grp.ws_tensor(grp.rank, low.gather_off + par * low.gather_par, (M, K))
        return out, gathered
    return out


def all_to_all_matmul(a_send: torch.Tensor, weight: torch.Tensor, kind=None, group: FiccoGroup | None = None,
                      out: torch.Tensor | None = None, stream=None, return_gathered: bool = False,
                      comm_agent: str | None = None):
    """EP dispatch -> expert GEMM with FiCCO overlap: C = all_to_all(A_send) @ W^T.

    ``a_send`` [G*R, K] holds G blocks of R token rows, block d addressed to rank d (uniform
    counts, as the reference's plans assume); W [N, K] is this rank's expert weight. Rows
    p*R.. of the result come from peer p's block for this rank. ``return_gathered`` also
    returns the dispatched tokens (a view into the group's double-buffered workspace).
    """
    grp = _default_group(group, None)
    _check_tensor("a_send", a_send)
    M, K = a_send.shape
    if M % grp.world:
        raise PlanError(f"send rows {M} must split into {grp.world} equal blocks")
    _check_tensor("weight", weight)
    R, N = M // grp.world, weight.shape[0]
    _check_call(grp, {"a_send": (a_send, None), "weight": (weight, (N, K))}, out, (M, N))
    plan, low, _ = prepare_a2a(grp, R, K, N, kind, comm_agent=_agent(comm_agent))
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a_send.device)
    _run(grp, plan, "a2a_gemm", a_send, weight, out, stream)
    if return_gathered:
        par = (grp.comm.epoch() - 1) & 1
        return out, grp.ws_tensor(grp.rank, low.gather_off + par * low.gather_par, (M, K))
    return out


def matmul_reduce_scatter(a: torch.Tensor, weight: torch.Tensor, kind=None, group: FiccoGroup | None = None,
                          out: torch.Tensor | None = None, stream=None, comm_agent: str | None = None):
    """C_shard = reduce_scatter_rows(A @ W^T). A [M, Kg], W [N, Kg] -> [M/G, N] (this rank's rows)."""
    grp = _default_group(group, None)
    _check_tensor("a", a)
    M, K = a.shape
    if M % grp.world:
        raise PlanError(f"rows {M} must split into {grp.world} equal output shards")
    _check_tensor("weight", weight)
    N = weight.shape[0]
    _check_call(grp, {"a": (a, None), "weight": (weight, (N, K))}, out, (M // grp.world, N))
    plan, _, _ = prepare_rs(grp, M, K, N, kind, comm_agent=_agent(comm_agent, "rs"))
    if out is None:
        out = torch.empty(M // grp.world, N, dtype=torch.bfloat16, device=a.device)
    _run(grp, plan, "gemm_rs", a, weight, out, stream)
    return out


def cp_kv_all_gather_qk(q: torch.Tensor, k_shard: torch.Tensor, kind=None, scale: float | None = None,
                        group: FiccoGroup | None = None, out: torch.Tensor | None = None, stream=None,
                        comm_agent: str | None = None):
    """S = scale * Q @ all_gather(K_shard)^T. Q [Tq, d], K_shard [Tkv/G, d] -> S [Tq, Tkv] (bf16).

    Scenario view: M = Tkv (gathered kv tokens), N = Tq, K = d.
    """
    grp = _default_group(group, None)
    _check_tensor("q", q)
    Tq, d = q.shape
    _check_tensor("k_shard", k_shard)
    Tkv = k_shard.shape[0] * grp.world
    _check_call(grp, {"q": (q, None), "k_shard": (k_shard, (Tkv // grp.world, d))}, out, (Tq, Tkv))
    agent = _agent(comm_agent)
    plan, low, kd = prepare_cp(grp, Tq, d, Tkv, kind, scale, comm_agent=agent)
    if _is_slot(grp, k_shard, low):  # zero-copy publish: the K shard already sits in its slot
        plan, _, _ = prepare_cp(grp, Tq, d, Tkv, kd, scale, comm_agent=agent, inplace=True)
    if out is None:
        out = torch.empty(Tq, Tkv, dtype=torch.bfloat16, device=q.device)
    _run(grp, plan, "cp_qk", q, k_shard, out, stream)
    return out

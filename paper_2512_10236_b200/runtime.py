"""ctypes binding of the C-ABI executor (include/ficco.h -> libficco_b200.so).

PyTorch is plumbing here: it owns caller buffers and streams, and
``torch.distributed`` exchanges CUDA-IPC handles of the symmetric workspaces.
Every compute call goes through the C library; there is no fallback — if the
library cannot be loaded or the device is not sm_100, calls raise.

Error mapping: FICCO_EINVAL -> ValueError, FICCO_ECUDA ->
RuntimeError, FICCO_ETIMEOUT -> DeadlockError (the reference's
engine.DeadlockError, engine.py:35), FICCO_ENODEV -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib
import threading

from .simulator import DeadlockError

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libficco_b200.so"

FICCO_WS_FLAG_WORDS = 16384
FICCO_WS_DATA_OFFSET = FICCO_WS_FLAG_WORDS * 4
FICCO_FLAG_BLOCK = 4096
FICCO_FLAG_RUN_LOCAL = 256
FICCO_FLAG_ABORT = FICCO_WS_FLAG_WORDS - 1
FICCO_FLAG_COUNTERS = 2048  # block-relative
FICCO_MAX_STREAMS = 16

OP_COPY, OP_SIGNAL, OP_NOTIFY, OP_WAIT, OP_WAIT_COUNTER, OP_BARRIER, OP_RECORD, OP_STREAM_WAIT, OP_REDUCE_MC = range(9)
FICCO_MAX_EVENTS = 64
BUF_NONE, BUF_A, BUF_B, BUF_C, BUF_WS, BUF_MC, BUF_MCV = 0, 1, 2, 3, 4, 5, 6
FICCO_HINT_A_EVICT_LAST, FICCO_HINT_CORE_COPIES, FICCO_HINT_B_EVICT_FIRST = 1, 2, 4  # ficco_plan_desc.hints
EPI_STORE, EPI_STORE_SIGNAL, EPI_REDUCE, EPI_STORE_REMOTE = 0, 1, 2, 3
TILE_M, TILE_N, TILE_K = 128, 256, 64
TILE_WIDTHS = (256, 224, 192, 160, 128)
MAX_RECV = 15

EXPORTED = (
    "ficco_abi_version", "ficco_last_error", "ficco_device_info", "ficco_ws_alloc", "ficco_ws_free",
    "ficco_ipc_handle_size", "ficco_ipc_get_handle", "ficco_ipc_open", "ficco_ipc_close",
    "ficco_comm_create", "ficco_comm_destroy", "ficco_comm_epoch", "ficco_comm_check", "ficco_comm_set_flags",
    "ficco_plan_create", "ficco_plan_destroy", "ficco_plan_run", "ficco_plan_run_parts",
    "ficco_gemm_bf16", "ficco_copy_batch", "ficco_plan_set_trace", "ficco_plan_info", "ficco_gemm_bf16_cfg", "ficco_occupy_sms",
    "ficco_timestamp", "ficco_watch_words", "ficco_ag_gemm", "ficco_a2a_gemm", "ficco_gemm_rs", "ficco_cp_qk",
    "ficco_plan_set_kernel_event", "ficco_mc_supported", "ficco_mc_create", "ficco_mc_export", "ficco_mc_import",
    "ficco_mc_add_device", "ficco_mc_bind", "ficco_mc_release", "ficco_comm_set_multicast", "ficco_mc_reduce_bf16",
)


class CopyOp(C.Structure):
    _fields_ = [("op", C.c_int32), ("peer", C.c_int32), ("flag", C.c_int32), ("src_buf", C.c_int32),
                ("dst_buf", C.c_int32), ("dst_peer", C.c_int32), ("src_off", C.c_int64), ("dst_off", C.c_int64),
                ("src_par", C.c_int64), ("dst_par", C.c_int64), ("width", C.c_int64), ("height", C.c_int64),
                ("src_pitch", C.c_int64), ("dst_pitch", C.c_int64), ("value", C.c_uint32),
                ("stream", C.c_int32)]


class Tile(C.Structure):
    _fields_ = [("a_row", C.c_int32), ("b_row", C.c_int32), ("c_row", C.c_int32), ("c_col", C.c_int32),
                ("recv_row", C.c_int32), ("rows", C.c_int16), ("cols", C.c_int16), ("flag", C.c_int16),
                ("fmask", C.c_uint16), ("kseg", C.c_int16), ("kstride", C.c_int16), ("mode", C.c_int16),
                ("chunk", C.c_int16), ("a_src", C.c_uint8), ("b_src", C.c_uint8), ("reserved", C.c_uint16)]


class Operand(C.Structure):
    _fields_ = [("buf", C.c_int32), ("pad", C.c_int32), ("off", C.c_int64), ("par", C.c_int64),
                ("rows", C.c_int64), ("ld", C.c_int64)]


class PlanDesc(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_tiles", C.c_int32), ("ops", C.POINTER(CopyOp)),
                ("tiles", C.POINTER(Tile)), ("a", Operand), ("b", Operand), ("c", Operand), ("part", Operand),
                ("recv", Operand), ("a2", Operand), ("b2", Operand), ("recv_slot", C.c_int64), ("k", C.c_int64),
                ("n_recv", C.c_int32),
                ("rs_flag0", C.c_int32), ("n_counters", C.c_int32), ("grid", C.c_int32), ("alpha", C.c_float),
                ("tile_n", C.c_int32), ("cta_group", C.c_int32), ("hints", C.c_int32), ("rs_target", C.c_int32),
                ("go_flag", C.c_int32)]


assert C.sizeof(CopyOp) == 96 and C.sizeof(Tile) == 40 and C.sizeof(Operand) == 40

_lib = None
_lock = threading.Lock()


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the C-ABI. Raises if the shared object is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = pathlib.Path(path or os.environ.get("FICCO_LIB_PATH") or LIB_PATH)
        if not p.exists():
            raise RuntimeError(f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(p))
        vp, i32, i64, sz = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
        sig = {
            "ficco_abi_version": ([], i32),
            "ficco_last_error": ([], C.c_char_p),
            "ficco_device_info": ([i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
            "ficco_ws_alloc": ([sz, C.POINTER(vp)], i32),
            "ficco_ws_free": ([vp], i32),
            "ficco_ipc_handle_size": ([], i32),
            "ficco_ipc_get_handle": ([vp, vp], i32),
            "ficco_ipc_open": ([vp, C.POINTER(vp)], i32),
            "ficco_ipc_close": ([vp], i32),
            "ficco_comm_create": ([i32, i32, C.POINTER(vp), sz, i32, C.POINTER(vp)], i32),
            "ficco_comm_destroy": ([vp], i32),
            "ficco_comm_epoch": ([vp, C.POINTER(C.c_uint32)], i32),
            "ficco_comm_check": ([vp, vp], i32),
            "ficco_comm_set_flags": ([vp, i32, i32, C.c_uint32, vp], i32),
            "ficco_plan_create": ([vp, C.POINTER(PlanDesc), C.POINTER(vp)], i32),
            "ficco_plan_destroy": ([vp], i32),
            "ficco_plan_run": ([vp, vp, vp, vp, vp], i32),
            "ficco_plan_run_parts": ([vp, vp, vp, vp, vp, i32, i32], i32),
            "ficco_ag_gemm": ([vp, vp, vp, vp, vp], i32),
            "ficco_a2a_gemm": ([vp, vp, vp, vp, vp], i32),
            "ficco_gemm_rs": ([vp, vp, vp, vp, vp], i32),
            "ficco_cp_qk": ([vp, vp, vp, vp, vp], i32),
            "ficco_gemm_bf16": ([vp, vp, vp, i64, i64, i64, C.c_float, i32, vp], i32),
            "ficco_gemm_bf16_cfg": ([vp, vp, vp, i64, i64, i64, C.c_float, i32, i32, i32, vp], i32),
            "ficco_copy_batch": ([C.POINTER(vp), C.POINTER(vp), C.POINTER(sz), sz, vp], i32),
            "ficco_occupy_sms": ([i64, vp], i32),
            "ficco_timestamp": ([vp, vp], i32),
            "ficco_watch_words": ([vp, i32, C.c_uint32, vp, i64, vp], i32),
            "ficco_plan_set_trace": ([vp, vp], i32),
            "ficco_plan_set_kernel_event": ([vp, vp], i32),
            "ficco_mc_supported": ([i32, C.POINTER(i32)], i32),
            "ficco_mc_create": ([sz, i32, C.POINTER(vp), C.POINTER(sz)], i32),
            "ficco_mc_export": ([vp, C.POINTER(i32)], i32),
            "ficco_mc_import": ([i32, sz, C.POINTER(vp)], i32),
            "ficco_mc_add_device": ([vp], i32),
            "ficco_mc_bind": ([vp, C.POINTER(vp), C.POINTER(vp)], i32),
            "ficco_mc_release": ([vp], i32),
            "ficco_comm_set_multicast": ([vp, vp, vp, sz], i32),
            "ficco_mc_reduce_bf16": ([vp, vp, i64, i64, i64, i64, vp], i32),
            "ficco_plan_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.ficco_abi_version() != 1:
            raise RuntimeError("libficco_b200 ABI mismatch")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load_library().ficco_last_error() or b"").decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -3:
        raise DeadlockError(msg)
    if rc == -4:
        raise NotImplementedError(msg)  # FICCO_ENODEV: the device / fabric lacks what the op needs
    raise RuntimeError(f"libficco_b200 error {rc}: {msg}")


def _stream_ptr(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Workspace:
    """A symmetric workspace buffer (flags + data) allocated by the library."""

    def __init__(self, nbytes: int):
        lib = load_library()
        ptr = C.c_void_p()
        check(lib.ficco_ws_alloc(nbytes, C.byref(ptr)))
        self.ptr = ptr.value
        self.nbytes = nbytes

    def ipc_handle(self) -> bytes:
        lib = load_library()
        buf = C.create_string_buffer(lib.ficco_ipc_handle_size())
        check(lib.ficco_ipc_get_handle(C.c_void_p(self.ptr), buf))
        return buf.raw

    def free(self) -> None:
        if self.ptr:
            check(load_library().ficco_ws_free(C.c_void_p(self.ptr)))
            self.ptr = None


def ipc_open(handle: bytes) -> int:
    out = C.c_void_p()
    check(load_library().ficco_ipc_open(C.create_string_buffer(handle, len(handle)), C.byref(out)))
    return out.value


def ipc_close(ptr: int) -> None:
    check(load_library().ficco_ipc_close(C.c_void_p(ptr)))


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All ranks' workspace IPC handles in rank order (plain bytes; any torch.distributed backend)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    handles: list = [None] * world
    dist.all_gather_object(handles, bytes(handle), group=group)
    if any(not isinstance(h, bytes) or len(h) != len(handle) for h in handles):
        raise RuntimeError("workspace handle exchange returned malformed handles")
    return handles


def multicast_supported(device: int = 0) -> bool:
    """Can this process create an NVLS multicast object on `device` (ficco_mc_supported)?"""
    ok = C.c_int()
    check(load_library().ficco_mc_supported(device, C.byref(ok)))
    return bool(ok.value)


class Multicast:
    """One rank's share of a group-wide NVLS multicast workspace (include/ficco.h setup order): rank 0
    creates the object and exports it as a POSIX fd; the peers duplicate that fd out of rank 0's process
    (pidfd_getfd; the ranks run as the same user on one node) and import it; every rank adds its device,
    meets the others, binds `nbytes` of its own HBM and maps the unicast and multicast views."""

    def __init__(self, nbytes: int, group=None):
        import torch.distributed as dist
        lib = load_library()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        h, mapped, fd = C.c_void_p(), C.c_size_t(), C.c_int(-1)
        err = None
        if rank == 0:
            try:
                check(lib.ficco_mc_create(nbytes, world, C.byref(h), C.byref(mapped)))
                check(lib.ficco_mc_export(h, C.byref(fd)))
            except Exception as exc:  # every rank must learn about it, or the peers would wait forever
                err = str(exc)
        info = [None] * world
        dist.all_gather_object(info, (os.getpid(), fd.value, mapped.value, err), group=group)
        pid0, fd0, mapped0, err0 = info[0]
        if err0:
            raise NotImplementedError(err0)
        if rank != 0:
            fd_local = _pidfd_getfd(pid0, fd0)
            check(lib.ficco_mc_import(fd_local, mapped0, C.byref(h)))
            os.close(fd_local)
        dist.barrier(group=group)
        check(lib.ficco_mc_add_device(h))
        dist.barrier(group=group)  # every device added before anyone binds memory
        uc, mc = C.c_void_p(), C.c_void_p()
        check(lib.ficco_mc_bind(h, C.byref(uc), C.byref(mc)))
        dist.barrier(group=group)
        if rank == 0:
            os.close(fd.value)
        self.handle, self.uc, self.va, self.nbytes = h.value, uc.value, mc.value, mapped0

    def release(self) -> None:
        if self.handle:
            check(load_library().ficco_mc_release(C.c_void_p(self.handle)))
            self.handle = None


def _pidfd_getfd(pid: int, fd: int) -> int:
    """Duplicate file descriptor `fd` of process `pid` into this process (Linux pidfd_open + pidfd_getfd)."""
    libc = C.CDLL(None, use_errno=True)
    pidfd = os.pidfd_open(pid)
    try:
        new = libc.syscall(438, pidfd, fd, 0)  # SYS_pidfd_getfd
        if new < 0:
            raise NotImplementedError(f"pidfd_getfd failed (errno {C.get_errno()}): cannot share the multicast "
                                      f"handle between ranks")
        return new
    finally:
        os.close(pidfd)


class Communicator:
    """One rank's view of G symmetric workspaces (+ its copy stream and epoch).

    ``Communicator.virtual(G, rank, nbytes)`` builds the single-process
    decomposition-only mode: the G-1 peers' workspaces are
    local allocations and cross-rank waits/notifies are satisfied locally.
    ``Communicator.from_process_group(nbytes, group)`` exchanges CUDA-IPC
    handles through ``torch.distributed`` (works for ranks on different GPUs
    of one node, and for several ranks sharing one GPU).
    """

    def __init__(self, rank: int, world: int, ws_ptrs: list[int], nbytes: int, virtual: bool,
                 owned: list[Workspace], opened: list[int]):
        lib = load_library()
        self._check_connections()
        arr = (C.c_void_p * world)(*ws_ptrs)
        h = C.c_void_p()
        check(lib.ficco_comm_create(rank, world, arr, nbytes, int(virtual), C.byref(h)))
        self.handle = h.value
        self.rank, self.world, self.nbytes, self.virtual = rank, world, nbytes, virtual
        self.ws_ptrs = list(ws_ptrs)
        self._owned, self._opened = owned, opened

    @staticmethod
    def _check_connections() -> None:
        try:
            n = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
        except ValueError:
            n = 8
        if n < FICCO_MAX_STREAMS + 1:
            import warnings
            warnings.warn(f"CUDA_DEVICE_MAX_CONNECTIONS={n}: copy chains may share a hardware queue with work "
                          f"that waits for the tile kernel (stalls until the flag timeout); set it to 32 before "
                          f"the first CUDA call", RuntimeWarning, stacklevel=3)

    @classmethod
    def virtual(cls, world: int, rank: int, nbytes: int) -> "Communicator":
        owned = [Workspace(nbytes) for _ in range(world)]
        return cls(rank, world, [w.ptr for w in owned], nbytes, True, owned, [])

    @classmethod
    def from_process_group(cls, nbytes: int, group=None) -> "Communicator":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        mine = Workspace(nbytes)
        handles = exchange_handles(mine.ipc_handle(), group)
        ptrs, opened = [], []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(mine.ptr)
            else:
                p = ipc_open(h)
                ptrs.append(p)
                opened.append(p)
        dist.barrier(group=group)
        return cls(rank, world, ptrs, nbytes, False, [mine], opened)

    @property
    def local_ws(self) -> int:
        return self.ws_ptrs[self.rank]

    def epoch(self) -> int:
        e = C.c_uint32()
        check(load_library().ficco_comm_epoch(C.c_void_p(self.handle), C.byref(e)))
        return e.value

    def check(self, stream=None) -> None:
        """Synchronise and raise DeadlockError if a kernel timed out on a flag."""
        check(load_library().ficco_comm_check(C.c_void_p(self.handle), C.c_void_p(_stream_ptr(stream))))

    def set_multicast(self, mc: "Multicast | None") -> None:
        """Attach (or detach) the group's NVLS multicast workspace (comm_agent = nvls plans)."""
        if mc is None:
            check(load_library().ficco_comm_set_multicast(C.c_void_p(self.handle), None, None, 0))
        else:
            check(load_library().ficco_comm_set_multicast(C.c_void_p(self.handle), C.c_void_p(mc.uc),
                                                          C.c_void_p(mc.va), mc.nbytes))

    def set_flags(self, first: int, count: int, value: int, stream=None) -> None:
        check(load_library().ficco_comm_set_flags(C.c_void_p(self.handle), first, count, value,
                                                  C.c_void_p(_stream_ptr(stream))))

    def close(self, between=None) -> None:
        """Destroy the communicator, unmap the peers' workspaces, then (after ``between()``,
        e.g. a process-group barrier) free the own ones."""
        if self.handle:
            load_library().ficco_comm_destroy(C.c_void_p(self.handle))
            self.handle = None
            for p in self._opened:
                ipc_close(p)
            self._opened = []
            if between is not None:
                between()
            for w in self._owned:
                w.free()
            self._owned = []

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """A lowered per-rank program bound to a communicator (ficco_plan_t)."""

    def __init__(self, comm: Communicator, desc: PlanDesc, ops: list[CopyOp], tiles: list[Tile]):
        lib = load_library()
        self._ops = (CopyOp * max(1, len(ops)))(*ops)
        self._tiles = (Tile * max(1, len(tiles)))(*tiles)
        desc.n_ops, desc.n_tiles = len(ops), len(tiles)
        desc.ops = C.cast(self._ops, C.POINTER(CopyOp))
        desc.tiles = C.cast(self._tiles, C.POINTER(Tile))
        h = C.c_void_p()
        check(lib.ficco_plan_create(C.c_void_p(comm.handle), C.byref(desc), C.byref(h)))
        self.handle, self.comm, self.desc = h.value, comm, desc
        self.n_ops, self.n_tiles = len(ops), len(tiles)

    def run(self, a, b, c, stream=None) -> None:
        """One execution replayed from the plan's CUDA graph (see ficco_plan_run)."""
        ptr = lambda t: C.c_void_p(0 if t is None else t.data_ptr())  # noqa: E731
        check(load_library().ficco_plan_run(C.c_void_p(self.handle), ptr(a), ptr(b), ptr(c),
                                            C.c_void_p(_stream_ptr(stream))))

    def run_op(self, op: str, a, b, c, stream=None) -> None:
        """The typed op entry point (ficco_ag_gemm / _a2a_gemm / _gemm_rs / _cp_qk): ficco_plan_run
        after the library checked that this plan was lowered for `op`."""
        ptr = lambda t: C.c_void_p(0 if t is None else t.data_ptr())  # noqa: E731
        check(getattr(load_library(), f"ficco_{op}")(C.c_void_p(self.handle), ptr(a), ptr(b), ptr(c),
                                                     C.c_void_p(_stream_ptr(stream))))

    def run_parts(self, a, b, c, stream=None, copies: bool = True, tiles: bool | int = True) -> None:
        """The same run enqueued directly on streams (no graph); halves selectable;
        tiles=2 serialises (copies, then kernel) for profilers."""
        ptr = lambda t: C.c_void_p(0 if t is None else t.data_ptr())  # noqa: E731
        check(load_library().ficco_plan_run_parts(C.c_void_p(self.handle), ptr(a), ptr(b), ptr(c),
                                                  C.c_void_p(_stream_ptr(stream)), int(copies), int(tiles)))

    def info(self) -> dict:
        n, g, s = C.c_int(), C.c_int(), C.c_int()
        check(load_library().ficco_plan_info(C.c_void_p(self.handle), C.byref(n), C.byref(g), C.byref(s)))
        return {"tiles": n.value, "grid": g.value, "streams": s.value}

    def set_trace(self, buf) -> None:
        """Attach a device int64 tensor of >= grid + 2*tiles entries (None detaches)."""
        self._trace = buf
        check(load_library().ficco_plan_set_trace(C.c_void_p(self.handle),
                                                  C.c_void_p(0 if buf is None else buf.data_ptr())))

    def set_kernel_event(self, event) -> None:
        """Record ``event`` (a torch.cuda.Event that has been recorded once, or None) on the launch
        stream right after the tile kernel of every later run: times the in-op kernel alone."""
        self._kernel_event = event
        check(load_library().ficco_plan_set_kernel_event(
            C.c_void_p(self.handle), C.c_void_p(0 if event is None else event.cuda_event)))

    def close(self) -> None:
        if self.handle:
            load_library().ficco_plan_destroy(C.c_void_p(self.handle))
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def gemm_bf16(a, b, out, alpha: float = 1.0, grid: int = 0, stream=None, tile_n: int = 0,
              cta_group: int = 0) -> None:
    """out[M,N] = alpha * a[M,K] @ b[N,K]^T with the tcgen05 tile kernel (no flags).

    tile_n / cta_group 0 = automatic (wave model; CTA pairs)."""
    m, k = a.shape
    n = b.shape[0]
    check(load_library().ficco_gemm_bf16_cfg(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                             C.c_void_p(out.data_ptr()), m, n, k, alpha, grid, tile_n, cta_group,
                                             C.c_void_p(_stream_ptr(stream))))


def timestamp(dst, stream=None) -> None:
    """dst (int64 CUDA tensor, one element) := %globaltimer ns, stream-ordered (trace op boundaries)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    check(load_library().ficco_timestamp(C.c_void_p(dst.data_ptr()), C.c_void_p(s.cuda_stream)))


def watch_words(words_ptr: int, n: int, want: int, out, timeout_ns: int = 10**9, stream=None) -> None:
    """Diagnostic arrival profile: out (int64 CUDA tensor, n + 1) := %globaltimer when each of the n device
    words at words_ptr first reads >= want (0 on timeout); out[n] = watcher start. Launch before a run."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    check(load_library().ficco_watch_words(C.c_void_p(words_ptr), n, want, C.c_void_p(out.data_ptr()), timeout_ns,
                                           C.c_void_p(s.cuda_stream)))

/*
 * ficco.h — C-ABI of the B200-native FiCCO executor (libficco_b200.so).
 *
 * The reference (overlap_sim 0.1.0, /root/reference/pkg) is a pure-Python
 * simulator: its only "executor" is engine.simulate(plan, machine, topo,
 * model) (/root/reference/pkg/src/overlap_sim/engine.py:117), which prices the
 * Transfer/Gather/Gemm/Scatter DAG produced by planner.build_plan
 * (/root/reference/pkg/src/overlap_sim/planner.py:409). This library is the
 * real executor that takes that slot: the Python layer lowers an
 * ExecutionPlan (per rank) into
 *   - a COPY PROGRAM run on a dedicated copy stream: copy-engine peer copies
 *     (cudaMemcpyAsync / cudaMemcpy2DAsync, no SMs; captured once into a CUDA
 *     graph per workspace parity) each followed by a copy-engine copy of a
 *     constant word that publishes the chunk's readiness flag (waits are
 *     cuStreamWaitValue32/64 stream memory operations), and
 *   - a TILE PROGRAM run by one persistent tcgen05/TMEM/TMA kernel on the
 *     compute stream whose producer warp gates each tile's TMA loads on those
 *     flags (no host round trip).
 * Each reference TaskSpec maps as follows:
 *   TransferSpec (planner.py:58-64)  -> FICCO_OP_COPY + FICCO_OP_SIGNAL
 *   GatherSpec   (planner.py:67-69)  -> folded: copies land in place
 *   GemmSpec     (planner.py:77-89)  -> ficco_tile entries (rows/col_block)
 *   ScatterSpec  (planner.py:72-74)  -> folded: epilogue writes C in place
 *   Task.deps    (planner.py:95-100) -> flag waits (copy stream or kernel)
 *
 * All device buffers are caller-owned except the symmetric workspace, which
 * the library allocates (ficco_ws_alloc) so it can be shared across ranks by
 * CUDA IPC. No C++ exception crosses this boundary: every entry point returns
 * 0 on success or a negative FICCO_E* code; ficco_last_error() gives the
 * thread-local message. Streams are cudaStream_t passed as void*.
 */
#ifndef FICCO_H_
#define FICCO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define FICCO_ABI_VERSION 1

/* status codes */
#define FICCO_OK 0
#define FICCO_EINVAL (-1)   /* bad argument (maps to ValueError / PlanError) */
#define FICCO_ECUDA (-2)    /* CUDA runtime/driver failure (RuntimeError) */
#define FICCO_ETIMEOUT (-3) /* a readiness flag never arrived (DeadlockError) */
#define FICCO_ENODEV (-4)   /* no sm_100 device */

/* Symmetric workspace layout: flag words first, data after FICCO_WS_DATA_OFFSET.
 * Flags are one-shot 0/1 words (constant values, so a lowered plan can be
 * replayed as a CUDA graph). Run r uses flag block (r & 1) — FICCO_FLAG_BLOCK
 * words each. Inside a block, words [0, FICCO_FLAG_RUN_LOCAL) are cross-rank
 * flags written by peers and reset by their consumer (FICCO_OP_WAIT); words
 * [FICCO_FLAG_RUN_LOCAL, FICCO_FLAG_BLOCK) are reset to 0 at the start of the
 * run that uses the block. */
#define FICCO_WS_FLAG_WORDS 16384
#define FICCO_WS_DATA_OFFSET (FICCO_WS_FLAG_WORDS * 4)
#define FICCO_FLAG_BLOCK 4096
#define FICCO_FLAG_RUN_LOCAL 256
#define FICCO_FLAG_COUNTERS 2048                   /* block-relative: per-unit tile counters (run-local) */
#define FICCO_FLAG_CONST_ONE 16320                 /* constant 0x01010101: source of flag-setting copies */
#define FICCO_FLAG_CONST_ZERO 16322                /* constant 8 zero bytes: source of flag resets */
#define FICCO_FLAG_ABORT (FICCO_WS_FLAG_WORDS - 1) /* kernel-side timeout indicator */
#define FICCO_WS_IDENTITY_OFF 40960                /* bytes: 64 x 64 bf16 identity (RS reduction operand) */
#define FICCO_MAX_STREAMS 16                       /* copy streams (parallel copy-engine chains) */

/* copy-program opcodes (executed in order on the copy stream) */
/* copy-program opcodes; ops with the same `stream` run in order on that copy
 * stream (one copy-engine chain); different streams run concurrently. Flags
 * are set by tiny copy-engine copies of a constant word (not by stream
 * write-value memops, which serialise across chains), so a flag lands right
 * behind the data it covers on the same engine. */
#define FICCO_OP_COPY 0         /* copy width x height bytes src -> dst (copy engine) */
#define FICCO_OP_SIGNAL 1       /* local flag[flag] := 1 (after everything before it on the stream);
                                   value > 1: words [flag, flag + value) at once (one memset) */
#define FICCO_OP_NOTIFY 2       /* flag[flag] of rank `peer` := 1 (remote write over NVLink) */
#define FICCO_OP_WAIT 3         /* wait until local flag[flag] != 0, then reset it (cross-rank flags) */
#define FICCO_OP_WAIT_COUNTER 4 /* wait until local counter[flag] >= value */
#define FICCO_OP_BARRIER 5      /* set byte `rank` of every rank's 8-byte barrier words at flag, wait for all, reset */
#define FICCO_OP_RECORD 6       /* record event slot `value` on the stream */
#define FICCO_OP_STREAM_WAIT 7  /* the stream waits for event slot `value` */
#define FICCO_OP_REDUCE_MC 8    /* comm_agent = nvls: dst (height x width bytes, dst_pitch) := the in-switch sum
                                   over every rank of the multicast view's rows at src (src_buf = MCV, src_pitch):
                                   multimem.ld_reduce.add.acc::f32 on bf16x2, one bf16 rounding */
#define FICCO_MAX_EVENTS 64

/* buffer ids */
#define FICCO_BUF_NONE 0
#define FICCO_BUF_A 1   /* call argument a */
#define FICCO_BUF_B 2   /* call argument b */
#define FICCO_BUF_C 3   /* call argument c */
#define FICCO_BUF_WS 4  /* symmetric workspace of rank `peer` (local rank for dst) */
#define FICCO_BUF_MC 5  /* comm_agent = nvls: this rank's memory bound to the multicast object (unicast VA) */
#define FICCO_BUF_MCV 6 /* comm_agent = nvls: the multicast VA of that object (loads reduce over every rank) */

/* epilogue modes of a tile */
#define FICCO_EPI_STORE 0        /* out[c] = bf16(alpha * acc) */
#define FICCO_EPI_STORE_SIGNAL 1 /* partial[c] = bf16(acc); counter[chunk] += 1 when the tile is stored */
#define FICCO_EPI_REDUCE 2       /* out[c] = bf16(acc + sum_j recv_j[...]) after rs flags of `chunk` */
#define FICCO_EPI_STORE_REMOTE 3 /* comm_agent = core GEMM -> RS: partial[c] = bf16(acc) stored straight into
                                    rank `chunk`'s receive slot for this rank (peer memory over NVLink, TMA),
                                    then that rank's flag word `recv_row` += 1 (release, system scope) */

typedef struct ficco_comm ficco_comm_t;
typedef struct ficco_plan ficco_plan_t;

typedef struct {
  int32_t op;       /* FICCO_OP_* */
  int32_t peer;     /* source rank of a COPY (pull) / target rank of a NOTIFY */
  int32_t flag;     /* flag / counter word index */
  int32_t src_buf;  /* FICCO_BUF_* */
  int32_t dst_buf;  /* FICCO_BUF_* (WS means the local workspace, or `dst_peer`'s when push) */
  int32_t dst_peer; /* -1: local; else rank whose workspace receives the bytes (push) */
  int64_t src_off, dst_off;     /* bytes from buffer base */
  int64_t src_par, dst_par;     /* added once per odd run (double-buffered workspaces) */
  int64_t width, height;        /* bytes per row, rows (height 1 = 1D copy) */
  int64_t src_pitch, dst_pitch; /* bytes between rows (2D) */
  uint32_t value;               /* WAIT_COUNTER threshold / event slot */
  int32_t stream;               /* copy stream index in [0, FICCO_MAX_STREAMS) */
} ficco_copy_op;

typedef struct {
  int32_t a_row;    /* row coordinate of the 128-row A box (TMA) */
  int32_t b_row;    /* row coordinate of the tile_n-row B box (TMA) */
  int32_t c_row;    /* first output row */
  int32_t c_col;    /* first output column */
  int32_t recv_row; /* REDUCE: row offset into every receive slot */
  int16_t rows;     /* valid output rows (<= 128; 0 = padding half of a CTA pair) */
  int16_t cols;     /* valid output columns (<= tile_n, multiple of 32) */
  int16_t flag;     /* base readiness flag gating the A/B loads (-1: none) */
  uint16_t fmask;   /* flags flag+i for every set bit i must all be set before the loads */
  int16_t kseg;     /* k-blocks (64 elements) per segment; segment s waits (flag + s*kstride, fmask) (0: off) */
  int16_t kstride;  /* flag stride between k segments */
  int16_t mode;     /* FICCO_EPI_* */
  int16_t chunk;    /* counter index (STORE_SIGNAL) or rs-flag group (REDUCE) */
  uint8_t a_src;    /* 0: A operand map; 1: alternate A map (a call argument, e.g. the local shard) */
  uint8_t b_src;    /* 0: B operand map; 1: alternate B map */
  uint16_t reserved;
} ficco_tile;

typedef struct {
  int32_t buf;      /* FICCO_BUF_* (WS = local workspace) */
  int32_t pad;
  int64_t off;      /* bytes */
  int64_t par;      /* extra bytes on odd runs */
  int64_t rows;     /* rows of the row-major bf16 matrix */
  int64_t ld;       /* elements between rows */
} ficco_operand;

typedef struct {
  int32_t n_ops;
  int32_t n_tiles;
  const ficco_copy_op* ops;
  const ficco_tile* tiles;
  ficco_operand a;    /* M x K, K contiguous (TMA box 128 x 64) */
  ficco_operand b;    /* N x K, K contiguous (TMA box tile_n x 64) */
  ficco_operand c;    /* output, bf16 */
  ficco_operand part; /* STORE_SIGNAL destination (RS partials) */
  ficco_operand recv; /* REDUCE sources: slot j at off + j*recv_slot (+par on odd runs) */
  ficco_operand a2;   /* alternate A source for tiles with a_src = 1 (FICCO_BUF_NONE: unused) */
  ficco_operand b2;   /* alternate B source for tiles with b_src = 1 */
  int64_t recv_slot;  /* bytes between receive slots */
  int64_t k;          /* reduction length in elements (multiple of 8) */
  int32_t n_recv;     /* receive slots summed by REDUCE tiles */
  int32_t rs_flag0;   /* first rs flag word (run-local); REDUCE waits flag[rs_flag0 + chunk*n_recv + j] */
  int32_t n_counters; /* counters [0, n_counters) reset to 0 before each run */
  int32_t grid;       /* persistent CTAs (0: one per SM) */
  float alpha;        /* epilogue scale (STORE) */
  int32_t tile_n;     /* tile width (UMMA N): 128, 160, 192, 224 or 256 (0: 256) */
  int32_t cta_group;  /* 1: one CTA per 128-row tile; 2: CTA pairs, tiles (2p, 2p+1) share b_row/c_col
                         and form one 256-row UMMA (0: 1) */
  int32_t hints;      /* FICCO_HINT_* bits (0: defaults) */
  int32_t rs_target;  /* REDUCE tiles wait flag[rs_flag0 + chunk*n_recv + j] >= rs_target (0: 1, one-shot flags;
                         STORE_REMOTE senders count their tiles into these words) */
  int32_t go_flag;    /* STORE_REMOTE tiles store only once local flag[go_flag] is set (the copy program's
                         DONE barrier: every owner has finished reading the previous run's slots); <= 0: none.
                         Remote slot of this rank on owner q: ws[q] + recv.off + slot*recv_slot, slot = rank
                         (rank < q) or rank - 1 (rank > q), recv.rows x recv.ld */
} ficco_plan_desc;

/* ficco_plan_desc.hints */
#define FICCO_HINT_A_EVICT_LAST 1 /* A is small and re-read by every column tile: keep it in L2 */
#define FICCO_HINT_CORE_COPIES 2  /* comm_agent = core: workspace-to-workspace transfers run as SM copy
                                     kernels (P2P loads/stores) instead of copy-engine memcpys */
#define FICCO_HINT_B_EVICT_FIRST 4 /* B is streamed once per tile column (column-major raster over row groups
                                      whose A slice is kept in L2): don't let it displace A */

int ficco_abi_version(void);
const char* ficco_last_error(void);

/* device / workspace / IPC */
int ficco_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);
int ficco_ws_alloc(size_t bytes, void** out);
int ficco_ws_free(void* ptr);
int ficco_ipc_handle_size(void);
int ficco_ipc_get_handle(void* ptr, void* out_handle);
int ficco_ipc_open(const void* handle, void** out);
int ficco_ipc_close(void* ptr);

/* communicator (replaces the interconnect model topology.Topology, overlap_sim/topology.py:20-47):
 * ws[r] = rank r's workspace as mapped in this process.
 * virtual_peers=1: a single process plays rank `rank` of `world`; peers'
 * workspaces are local allocations and cross-rank waits/notifies are
 * satisfied locally (decomposition-only mode). */
int ficco_comm_create(int rank, int world, void* const* ws, size_t ws_bytes, int virtual_peers,
                      ficco_comm_t** out);
int ficco_comm_destroy(ficco_comm_t* comm);
int ficco_comm_epoch(ficco_comm_t* comm, uint32_t* runs); /* runs started so far */
/* blocks until all work of the communicator finished; FICCO_ETIMEOUT if a kernel hit its flag timeout
 * (raised as the reference's engine.DeadlockError, overlap_sim/engine.py:35-36, 231-236) */
int ficco_comm_check(ficco_comm_t* comm, void* stream);
/* set local flag words [first, first+count) (absolute word index) to value, stream-ordered on `stream` */
int ficco_comm_set_flags(ficco_comm_t* comm, int first, int count, uint32_t value, void* stream);

/* plans: one rank's share of planner.build_plan's ExecutionPlan (overlap_sim/planner.py:409, DAG payloads
 * planner.py:58-113), lowered to a copy program + tile list by paper_2512_10236_b200/lowering.py */
int ficco_plan_create(ficco_comm_t* comm, const ficco_plan_desc* desc, ficco_plan_t** out);
int ficco_plan_destroy(ficco_plan_t* plan);
/* One execution (executes what engine.simulate prices, overlap_sim/engine.py:117-297), replayed from a
 * CUDA graph (one per flag/workspace parity,
 * instantiated on first use, kernel/copy nodes re-pointed when a/b/c change):
 * run-local flag reset, copy program on the copy streams and the tile kernel,
 * all joined into `stream`. Advances the comm's run counter. Non-blocking. */
int ficco_plan_run(ficco_plan_t* plan, const void* a, const void* b, void* c, void* stream);
/* Same semantics enqueued directly on streams (no graph); run_copies / run_tiles
 * select the halves (calibration of the loss model's DIL/CIL tables, overlap_sim/lossmodel.py:85-108,
 * engine.base_duration engine.py:76-103; a tile half alone only terminates if
 * its flags are satisfied). run_tiles = 2: serialised — the kernel launches after
 * the whole copy program (for kernel profilers that serialise work). */
int ficco_plan_run_parts(ficco_plan_t* plan, const void* a, const void* b, void* c, void* stream,
                         int run_copies, int run_tiles);

/* Typed op entry points (the overlapped-op boundary of SURVEY.md §8b): ficco_plan_run with the
 * call arguments named for the op, after checking that the plan was lowered for that op
 * (FICCO_EINVAL otherwise). bf16 row-major operands; W in nn.Linear layout [N, K].
 *   ficco_ag_gemm   C [G*R, N] = all_gather(A_shard [R, K]) @ W^T
 *   ficco_a2a_gemm  C [G*R, N] = all_to_all(A_send [G*R, K]) @ W^T   (block d of A_send -> rank d)
 *   ficco_gemm_rs   C_shard [M/G, N] = reduce_scatter_rows(A [M, Kg] @ W^T)
 *   ficco_cp_qk     S [Tq, Tkv] = alpha * Q [Tq, d] @ all_gather(K_shard [Tkv/G, d])^T */
int ficco_ag_gemm(ficco_plan_t* plan, const void* a_shard, const void* w, void* c, void* stream);
int ficco_a2a_gemm(ficco_plan_t* plan, const void* a_send, const void* w, void* c, void* stream);
int ficco_gemm_rs(ficco_plan_t* plan, const void* a, const void* w, void* c_shard, void* stream);
int ficco_cp_qk(ficco_plan_t* plan, const void* q, const void* k_shard, void* scores, void* stream);

/* Optional measured timeline: buf (device, u64) receives %globaltimer ns stamps —
 * [0, grid) CTA start, then per tile t {2t: flags satisfied / loads start,
 * 2t+1: tile stored} at offset grid. NULL disables. Rebuilds the plan's graphs. */
int ficco_plan_set_trace(ficco_plan_t* plan, void* buf);
int ficco_plan_info(ficco_plan_t* plan, int* n_tiles, int* grid, int* n_streams);
/* Optional: record `event` (a cudaEvent_t) on the caller's stream right after the tile kernel in
 * every later ficco_plan_run, so (event before the call -> event) times the in-op kernel alone
 * (bench.py's roofline). NULL detaches. Not available with FICCO_KERNEL_IN_GRAPH=1. */
int ficco_plan_set_kernel_event(ficco_plan_t* plan, void* event);

/* NVLS (NVLink SHARP) multicast for comm_agent = nvls GEMM -> reduce-scatter: each rank stores its whole
 * partial into memory bound to one multicast object; an owner reads its rows through the multicast VA with
 * multimem.ld_reduce, so NVSwitch returns the sum over every rank. Setup (collective, in order):
 * rank 0 ficco_mc_create -> ficco_mc_export (POSIX fd, passed to the peers) -> peers ficco_mc_import ->
 * every rank ficco_mc_add_device -> barrier -> every rank ficco_mc_bind -> ficco_comm_set_multicast.
 * Where the driver cannot create multicast objects (no NVSwitch fabric access) these return FICCO_ENODEV
 * with the driver's reason. */
int ficco_mc_supported(int device, int* supported); /* 1 only if a multicast object can really be created */
int ficco_mc_create(size_t bytes, int n_devices, void** mc, size_t* mapped_bytes);
int ficco_mc_export(void* mc, int* fd);
int ficco_mc_import(int fd, size_t mapped_bytes, void** mc);
int ficco_mc_add_device(void* mc);
int ficco_mc_bind(void* mc, void** uc_va, void** mc_va); /* back the object with this device's memory, map both */
int ficco_mc_release(void* mc);                        /* unmap, unbind, free (after every rank stopped using it) */
int ficco_comm_set_multicast(ficco_comm_t* comm, void* uc_va, void* mc_va, size_t bytes);
/* dst[rows x cols bf16, ld_dst] := sum over the multicast object's devices of src[.., ld_src] (src = mc VA) */
int ficco_mc_reduce_bf16(const void* mc_src, void* dst, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
                         void* stream);

/* stand-alone primitives (calibration, benchmarks) */
int ficco_gemm_bf16(const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k, float alpha,
                    int grid, void* stream);
/* tile_n 0 / cta_group 0: automatic (waves x (width + 512) model, CTA pairs); the GEMM task price
 * flops / effective_flops of engine.py:86-93 measured instead of modelled */
int ficco_gemm_bf16_cfg(const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k, float alpha,
                        int grid, int tile_n, int cta_group, void* stream);
int ficco_copy_batch(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t count,
                     void* stream);
/* Occupy every SM (one CTA per SM holding all registers and shared memory) for `ns`
 * nanoseconds: copies issued meanwhile progress only if a copy engine executes them
 * (copy-engine vs SM-copy-kernel probe; CIL calibration). */
int ficco_occupy_sms(int64_t ns, void* stream);
/* Write the %globaltimer (ns, same clock as ficco_plan_set_trace stamps) to device u64 *dst,
 * stream-ordered: marks an op's start/end on the tile kernel's timeline. */
int ficco_timestamp(void* dst, void* stream);
/* Diagnostic: one CTA polls device words[0..n) until each is >= want and writes the
 * %globaltimer of its arrival to u64 out[i] (0 after timeout_ns); out[n] = watcher start.
 * Gives the copy program's per-flag arrival profile (launch it before the run). */
int ficco_watch_words(const void* words, int n, uint32_t want, void* out, int64_t timeout_ns, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* FICCO_H_ */

// libficco_b200: C-ABI executor for lowered FiCCO plans on B200 (sm_100a).
//
// Host side of the executor declared in include/ficco.h. Responsibilities:
//   * symmetric workspace + CUDA IPC plumbing (ranks exchange handles in Python),
//   * the copy program: one copy-engine copy per chunk (cudaMemcpyAsync 1D /
//     cudaMemcpy2DAsync for 2D slabs) on per-peer copy streams, readiness flags
//     written by tiny copy-engine copies of a constant word right behind the data,
//     waits as stream memory operations (cuStreamWaitValue32/64) — no SMs, no host
//     round trips; the whole program is captured once per workspace parity into a
//     CUDA graph and replayed. (ficco_copy_batch issues a list of copies, one
//     cudaMemcpyAsync each, for calibration probes; the plans do not use it.)
//   * the tile program: TMA descriptors + one persistent tcgen05 kernel launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ficco.h"
#include "copy_kernel.cuh"
#include "multicast.cuh"
#include "tile_kernel.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(FICCO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +        \
                                   std::to_string(__LINE__));                                     \
  } while (0)

#define CKD(call)                                                                                 \
  do {                                                                                            \
    CUresult r_ = (call);                                                                         \
    if (r_ != CUDA_SUCCESS)                                                                       \
      return fail(FICCO_ECUDA, std::string(#call) + ": CUresult " + std::to_string(int(r_)) + " @" + \
                                   std::to_string(__LINE__));                                     \
  } while (0)

// ---------------------------------------------------------------- driver entry points
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

struct Driver {
  PFN_encodeTiled encode = nullptr;
  PFN_writeValue32 write32 = nullptr;
  PFN_waitValue32 wait32 = nullptr;
  PFN_waitValue64 wait64 = nullptr;
  bool ok = false;
};

int get_driver(Driver** out) {
  static Driver d;
  static std::once_flag once;
  static int status = 0;
  static std::string err;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) -> bool {
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
      return e == cudaSuccess && q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    bool ok = get("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&d.encode)) &&
              get("cuStreamWriteValue32", reinterpret_cast<void**>(&d.write32)) &&
              get("cuStreamWaitValue32", reinterpret_cast<void**>(&d.wait32)) &&
              get("cuStreamWaitValue64", reinterpret_cast<void**>(&d.wait64));
    d.ok = ok;
    if (!ok) {
      status = FICCO_ECUDA;
      err = "could not resolve CUDA driver entry points (no driver / no GPU?)";
    }
  });
  if (status != 0) return fail(status, err);
  *out = &d;
  return 0;
}

// bf16 store boxes of 32 rows x box_cols (64: SWIZZLE_128B, 32: SWIZZLE_64B) — the epilogue's staging layouts.
int encode_store_map(Driver* drv, CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                     int box_cols) {
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0 || (ld * 2) % 16 != 0)
    return fail(FICCO_EINVAL, "output not 16-byte aligned");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  cuuint32_t box[2] = {cuuint32_t(box_cols), 32};
  cuuint32_t estr[2] = {1, 1};
  CKD(drv->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return 0;
}

int encode_bf16_2d(Driver* drv, CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                   int box_rows) {
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return fail(FICCO_EINVAL, "operand base not 16-byte aligned");
  if ((ld * 2) % 16 != 0) return fail(FICCO_EINVAL, "operand row pitch not a multiple of 16 bytes");
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  cuuint32_t box[2] = {cuuint32_t(ficco::BK), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CKD(drv->encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return 0;
}

// Epilogue staging buffers per warp: short-K tile programs (a handful of k-blocks per tile,
// e.g. C4's d = 128) are paced by the epilogue's TMEM reads and stores, so they keep 3 bulk
// stores in flight per warp; long-K programs are MMA-bound and keep the smem for stages.
int epi_bufs_for(int64_t k) { return k <= 384 ? 3 : 1; }

// What a lowered program computes, from its structure: GEMM -> RS programs carry partial /
// reduce tiles; gather programs read a workspace operand (A: AG and all-to-all dispatch; B: the
// CP KV gather); anything else is a plain GEMM.
enum { ROLE_PLAIN = 0, ROLE_GATHER_A = 1, ROLE_GATHER_B = 2, ROLE_REDUCE_SCATTER = 3 };
int plan_role(const ficco_plan_desc& d) {
  for (int i = 0; i < d.n_tiles; ++i)
    if (d.tiles[i].mode != FICCO_EPI_STORE) return ROLE_REDUCE_SCATTER;
  if (d.b.buf == FICCO_BUF_WS) return ROLE_GATHER_B;
  if (d.a.buf == FICCO_BUF_WS) return ROLE_GATHER_A;
  return ROLE_PLAIN;
}

// Rows per raster group of the plain GEMM (lowering.raster for the ops): row-major tiles
// (M outer) while B [N, K] fits in L2 — every B tile then comes from L2; short-K, store-bound
// shapes sweep the whole M extent per column block (each B tile read from HBM once, the small A
// stays in L2); a B too large for L2 goes column-major over row groups whose A slice fits.
// Rows per raster group of the plain GEMM (lowering.raster mirrors it). A weight up to 32 MiB stays
// L2-resident under a row-major raster (C2). A larger one would be re-read from HBM by every wave
// (C3's 59 MiB W: 0.86 GB of DRAM reads for 176 MB of operands), so rows go in groups whose A slice
// (<= 32 MiB, pinned evict_last) stays in L2 while each group sweeps N: C3 0.40 GB, 2-3 % faster
// (profiles/r02_experiments/c3_raster_ab.json). ceil(m / budget) groups, balanced.
int64_t raster_rows(int64_t m, int64_t n, int64_t k, int64_t mstep) {
  if (epi_bufs_for(k) > 1) return m;
  if (n * k * 2 <= (int64_t(32) << 20)) return mstep;
  const int64_t budget = std::max<int64_t>(mstep, (int64_t(32) << 20) / (k * 2) / mstep * mstep);
  const int64_t groups = (m + budget - 1) / budget;
  return ((m + groups - 1) / groups + mstep - 1) / mstep * mstep;
}

// Resolve the (tile width, CTA group, staging buffers) instantiation: entry point, dynamic smem,
// B box rows.
int kernel_for(int tn, int cg, int eb, const void** fn, int* smem, int* b_rows, int* stages = nullptr) {
#define FICCO_CASE(T, G, E)                                                  \
  if (tn == T && cg == G && eb == E) {                                       \
    *fn = reinterpret_cast<const void*>(ficco::tile_gemm_kernel<T, G, E>);   \
    *smem = ficco::TileCfg<T, G, E>::SMEM_BYTES;                             \
    *b_rows = ficco::TileCfg<T, G, E>::B_ROWS;                               \
    if (stages) *stages = ficco::TileCfg<T, G, E>::STAGES;                   \
    return 0;                                                                \
  }
  FICCO_FOR_EACH_CFG(FICCO_CASE)
#undef FICCO_CASE
  return fail(FICCO_EINVAL, "unsupported tile config " + std::to_string(tn) + "x" + std::to_string(cg));
}

int configure_kernels(int dev) {
  // per device: cudaFuncSetAttribute is per (function, device) and processes may drive several GPUs
  static std::mutex mu;
  static uint64_t configured = 0;  // bit d: device d done
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 64 && (configured >> dev) & 1u) return 0;
  if (const char* env = getenv("FICCO_L2_PERSIST_MB")) {  // L2 set-aside for evict_last lines (experiments)
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(atoll(env)) << 20));
  }
#define FICCO_CFG(T, G, E)                                                                              \
  CK(cudaFuncSetAttribute(ficco::tile_gemm_kernel<T, G, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                          ficco::TileCfg<T, G, E>::SMEM_BYTES));                                        \
  {                                                                                                     \
    cudaFuncAttributes fa;                                                                              \
    CK(cudaFuncGetAttributes(&fa, ficco::tile_gemm_kernel<T, G, E>));                                   \
    if (fa.numRegs * ficco::NUM_THREADS > 65536 - ficco::COPY_RESERVE_REGS)                          \
      return fail(FICCO_ECUDA, "tile kernel register use leaves no room for copy kernels");      \
  }
  FICCO_FOR_EACH_CFG(FICCO_CFG)
#undef FICCO_CFG
  if (dev >= 0 && dev < 64) configured |= uint64_t(1) << dev;
  return 0;
}

}  // namespace

namespace ficco {
// Spin for `ns` with every register and shared-memory byte of the SM taken (launch 1 CTA x 1024
// threads per SM with the opt-in smem maximum): nothing else can be resident meanwhile.
__global__ void __launch_bounds__(1024, 1) occupy_kernel(int64_t ns) {
  extern __shared__ uint8_t occ_smem[];
  const unsigned long long t0 = globaltimer();
  if (threadIdx.x == 0) occ_smem[0] = 1;
  while (int64_t(globaltimer() - t0) < ns) __nanosleep(256);
}
// One %globaltimer stamp, stream-ordered (op-boundary marks for the tile kernel's trace).
__global__ void stamp_kernel(unsigned long long* dst) { *dst = globaltimer(); }
// Arrival profile of readiness words (diagnostic): thread i polls words[i] until it is >= want and
// writes the %globaltimer of that moment to out[i] (0 on timeout); out[n] = the watcher's own start.
__global__ void watch_kernel(const uint32_t* words, int n, uint32_t want, unsigned long long* out,
                             int64_t timeout_ns) {
  const unsigned long long t0 = globaltimer();
  if (threadIdx.x == 0) out[n] = t0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long t = 0;
    for (;;) {
      uint32_t v;
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(words + i) : "memory");
      const unsigned long long now = globaltimer();
      if (v >= want) { t = now; break; }
      if (int64_t(now - t0) > timeout_ns) break;
    }
    out[i] = t;
  }
}
}  // namespace ficco

struct ficco_comm {
  int rank = 0, world = 1, device = 0, sms = 0;
  bool virt = false;
  size_t ws_bytes = 0;
  std::vector<uint8_t*> ws;  // per rank, mapped into this process
  uint32_t runs = 0;         // runs started; run r uses flag block / workspace parity r & 1
  cudaStream_t copy[FICCO_MAX_STREAMS] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[FICCO_MAX_STREAMS] = {};
  cudaEvent_t ev_pool[FICCO_MAX_EVENTS] = {};
  // host-mapped copy of the abort word: the tile kernel raises it with the device word when a flag
  // wait times out, so every later run can refuse a poisoned communicator without a device sync
  uint32_t* host_abort = nullptr;
  uint32_t* dev_host_abort = nullptr;
  // comm_agent = nvls: this rank's memory bound to the group's multicast object (unicast VA) and the
  // multicast VA (ficco_comm_set_multicast); null when the group has none
  uint8_t* mc_uc = nullptr;
  uint8_t* mc_va = nullptr;
  size_t mc_bytes = 0;
  Driver* drv = nullptr;
  uint32_t* flags(int r) { return reinterpret_cast<uint32_t*>(ws[r]); }
  uint32_t* block(int r, uint32_t parity) { return flags(r) + parity * FICCO_FLAG_BLOCK; }
};

struct GraphInst {
  cudaGraph_t graph = nullptr;  // kept alive: node handles index into it for exec updates
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t kernel = nullptr;
  std::vector<std::pair<cudaGraphNode_t, int>> user_copies;
  std::vector<std::pair<cudaGraphNode_t, int>> user_reduces;  // REDUCE_MC kernel nodes writing a call argument
  const void* a = nullptr;
  const void* b = nullptr;
  void* c = nullptr;
};

struct ficco_plan {
  ficco_comm* comm = nullptr;
  std::vector<ficco_copy_op> ops;
  ficco_tile* d_tiles = nullptr;
  int n_tiles = 0;
  int n_streams = 0;
  bool user_copies = false;  // some copy touches a call argument (kept out of the graph)
  cudaGraphNode_t captured_kernel = nullptr;
  std::vector<std::pair<cudaGraphNode_t, int>> captured_copies;  // (node, op index) touching call arguments
  std::vector<std::pair<cudaGraphNode_t, int>> captured_reduces;
  unsigned long long* trace = nullptr;  // optional device timeline buffer
  cudaEvent_t kernel_event = nullptr;   // optional: recorded on the launch stream right after the tile kernel
  // Kernel parameters of the last direct launch per workspace parity: reused while the call arguments,
  // the trace buffer and the launch-time knobs are unchanged (encoding the ~10-40 TMA descriptors is
  // most of an op's host time)
  struct ParamCache {
    bool valid = false;
    const void* a = nullptr;
    const void* b = nullptr;
    void* c = nullptr;
    unsigned long long* trace = nullptr;
    std::string knobs;
    int grid = 0;
    ficco::TileParams prm;
  };
  ParamCache pcache[2];
  bool concurrent = true;               // false: copies complete before the kernel starts (profilers)
  // Default: the tile kernel is launched directly on the caller's stream, THEN the copy-only
  // graph on a side stream (kernel first: it is queued before any of the graph's stream-wait
  // nodes exists, so a blocked wait — RS counter, cross-rank barrier — can never hold back the
  // kernel that satisfies it). Saves ~2 us of graph-launch latency before the first CTA (C2
  // 167.9 -> 165.9 us); every GPU test, multi-process ones included, passes in both modes.
  // FICCO_KERNEL_IN_GRAPH=1 makes the kernel a node of the run's graph instead.
  bool kernel_in_graph = false;
  bool counter_waits = false;           // the copy program waits on tile counters (RS dma pushes)
  int tile_n = 256;                     // tile width (UMMA N)
  int epi_bufs = 1;                     // epilogue staging buffers per warp (epi_bufs_for)
  bool has_remote = false;              // STORE_REMOTE tiles: peers' receive slots are TMA store targets
  int role = 0;                         // ROLE_* (which typed entry point may run it)
  int cta_group = 1;                    // 1: one CTA per tile; 2: CTA pair (cluster of 2, UMMA M = 256)
  ficco_plan_desc desc{};
  GraphInst graph[2];
};

namespace {

int resolve(ficco_comm* c, uint32_t parity, int buf, int peer, int64_t off, int64_t par, const void* a,
            const void* b, void* cc, uint8_t** out) {
  uint8_t* base = nullptr;
  switch (buf) {
    case FICCO_BUF_A: base = (uint8_t*)a; break;
    case FICCO_BUF_B: base = (uint8_t*)b; break;
    case FICCO_BUF_C: base = (uint8_t*)cc; break;
    case FICCO_BUF_WS:
      if (peer < 0) peer = c->rank;
      if (peer >= c->world) return fail(FICCO_EINVAL, "workspace peer out of range");
      base = c->ws[peer];
      break;
    case FICCO_BUF_MC: base = c->mc_uc; break;
    case FICCO_BUF_MCV: base = c->mc_va; break;
    default: return fail(FICCO_EINVAL, "bad buffer id " + std::to_string(buf));
  }
  if (!base) return fail(FICCO_EINVAL, "null buffer for id " + std::to_string(buf));
  *out = base + off + (parity ? par : 0);
  return 0;
}

bool is_user(int buf) { return buf == FICCO_BUF_A || buf == FICCO_BUF_B || buf == FICCO_BUF_C; }

int core_copy_ctas() {
  static const int n = [] {
    const char* env = getenv("FICCO_CORE_COPY_CTAS");
    const int v = env ? atoi(env) : 0;
    return v > 0 ? v : 32;
  }();
  return n;
}

int enqueue_copy(ficco_comm* cm, uint32_t parity, const ficco_copy_op& op, const void* a, const void* b, void* c,
                 cudaStream_t s, bool core) {
  uint8_t *src, *dst;
  int r = resolve(cm, parity, op.src_buf, op.peer, op.src_off, op.src_par, a, b, c, &src);
  if (r) return r;
  r = resolve(cm, parity, op.dst_buf, op.dst_peer, op.dst_off, op.dst_par, a, b, c, &dst);
  if (r) return r;
  const int64_t height = op.height <= 1 ? 1 : op.height;
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | uint64_t(op.width) |
                         (height > 1 ? uint64_t(op.src_pitch | op.dst_pitch) : 0)) & 15) == 0;
  if (core && op.src_buf == FICCO_BUF_WS && op.dst_buf == FICCO_BUF_WS && aligned) {
    // comm_agent = core: the transfer runs on SMs (P2P loads / stores), next to the tile kernel
    const int64_t vecs = op.width / 16 * height;
    const int64_t need = (vecs + ficco::COPY_THREADS * ficco::COPY_UNROLL - 1) / (ficco::COPY_THREADS * ficco::COPY_UNROLL);
    const int grid = int(need < core_copy_ctas() ? (need > 0 ? need : 1) : core_copy_ctas());
    ficco::sm_copy_kernel<<<grid, ficco::COPY_THREADS, 0, s>>>(dst, src, op.width, height,
                                                               height > 1 ? op.src_pitch : op.width,
                                                               height > 1 ? op.dst_pitch : op.width);
    CK(cudaGetLastError());
    return 0;
  }
  if (op.height <= 1) {
    CK(cudaMemcpyAsync(dst, src, size_t(op.width), cudaMemcpyDefault, s));
  } else {
    CK(cudaMemcpy2DAsync(dst, size_t(op.dst_pitch), src, size_t(op.src_pitch), size_t(op.width),
                         size_t(op.height), cudaMemcpyDefault, s));
  }
  return 0;
}

// One run enqueued on `s` + the copy streams (also used under stream capture to build the graph).
int enqueue_run(ficco_plan* p, uint32_t parity, const void* a, const void* b, void* c, cudaStream_t s,
                bool copies, bool tiles, int (*launch)(ficco_plan*, uint32_t, const void*, const void*, void*,
                                                      cudaStream_t)) {
  ficco_comm* cm = p->comm;
  // Run-local flags and counters of THIS run's block were cleared during the previous run;
  // clear the other block for the next run on a side stream, concurrently with this one.
  // (Runs r-1 and r+1 share that block; r-1 is complete, and peers only write its run-local
  // words after the owner's next DONE/PUB barrier, which follows this memset.)
  cudaStream_t side = cm->copy[FICCO_MAX_STREAMS - 1];
  CK(cudaEventRecord(cm->ev_fork, s));
  CK(cudaStreamWaitEvent(side, cm->ev_fork, 0));
  CK(cudaMemsetAsync(cm->block(cm->rank, parity ^ 1u) + FICCO_FLAG_RUN_LOCAL, 0,
                     4 * size_t(FICCO_FLAG_BLOCK - FICCO_FLAG_RUN_LOCAL), side));
  const bool fork = copies && p->n_streams > 0;
  if (fork)
    for (int i = 0; i < p->n_streams; ++i) CK(cudaStreamWaitEvent(cm->copy[i], cm->ev_fork, 0));
  const bool serialize = tiles && !p->concurrent;  // profiler mode: copies first, then the kernel
  if (tiles && !serialize) {
    int r = launch(p, parity, a, b, c, s);
    if (r) return r;
  }
  if (fork) {
    for (const ficco_copy_op& op : p->ops) {
      cudaStream_t cs = cm->copy[op.stream];
      switch (op.op) {
        case FICCO_OP_COPY: {
          int r = enqueue_copy(cm, parity, op, a, b, c, cs, (p->desc.hints & FICCO_HINT_CORE_COPIES) != 0);
          if (r) return r;
          if (is_user(op.src_buf) || is_user(op.dst_buf)) {  // remember it for graph re-pointing
            cudaStreamCaptureStatus st;
            CK(cudaStreamIsCapturing(cs, &st));
            if (st == cudaStreamCaptureStatusActive) {
              if (op.height > 1) return fail(FICCO_EINVAL, "2D copies of call arguments are not supported");
              const cudaGraphNode_t* deps = nullptr;
              size_t nd = 0;
              CK(cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &deps, &nd));
              if (nd != 1) return fail(FICCO_ECUDA, "graph capture: copy node not found");
              p->captured_copies.push_back({deps[0], int(&op - p->ops.data())});
            }
          }
          break;
        }
        case FICCO_OP_SIGNAL:
          if (op.value > 1)  // a run of words (e.g. virtual peers' pre-landed partials): 0x01010101 each
            CK(cudaMemsetAsync(cm->block(cm->rank, parity) + op.flag, 0x01, 4 * size_t(op.value), cs));
          else
            CK(cudaMemcpyAsync(cm->block(cm->rank, parity) + op.flag, cm->flags(cm->rank) + FICCO_FLAG_CONST_ONE, 4,
                               cudaMemcpyDeviceToDevice, cs));
          break;
        case FICCO_OP_NOTIFY:
          if (op.peer < 0 || op.peer >= cm->world) return fail(FICCO_EINVAL, "notify peer out of range");
          if (!cm->virt)
            CK(cudaMemcpyAsync(cm->block(op.peer, parity) + op.flag, cm->flags(cm->rank) + FICCO_FLAG_CONST_ONE, 4,
                               cudaMemcpyDefault, cs));
          break;
        case FICCO_OP_WAIT:
          if (!cm->virt) {
            uint32_t* f = cm->block(cm->rank, parity) + op.flag;
            CKD(cm->drv->wait32(cs, CUdeviceptr(f), 1u, CU_STREAM_WAIT_VALUE_GEQ));
            CK(cudaMemcpyAsync(f, cm->flags(cm->rank) + FICCO_FLAG_CONST_ZERO, 4, cudaMemcpyDeviceToDevice, cs));
          }
          break;
        case FICCO_OP_WAIT_COUNTER:
          CKD(cm->drv->wait32(cs, CUdeviceptr(cm->block(cm->rank, parity) + FICCO_FLAG_COUNTERS + op.flag),
                              op.value, CU_STREAM_WAIT_VALUE_GEQ));
          break;
        case FICCO_OP_BARRIER: {
          if (cm->virt) break;
          if (op.flag % 2) return fail(FICCO_EINVAL, "barrier word must be 8-byte aligned");
          const int nwords = (cm->world + 7) / 8;
          const uint8_t* one = reinterpret_cast<const uint8_t*>(cm->flags(cm->rank) + FICCO_FLAG_CONST_ONE);
          for (int q = 0; q < cm->world; ++q) {  // byte `rank` of everyone's barrier (own included)
            uint8_t* dst = reinterpret_cast<uint8_t*>(cm->block(q, parity) + op.flag) + cm->rank;
            CK(cudaMemcpyAsync(dst, one, 1, cudaMemcpyDefault, cs));
          }
          uint64_t* mine = reinterpret_cast<uint64_t*>(cm->block(cm->rank, parity) + op.flag);
          for (int w = 0; w < nwords; ++w) {
            uint64_t want = 0;
            for (int q = 8 * w; q < cm->world && q < 8 * w + 8; ++q) want |= uint64_t(1) << (8 * (q - 8 * w));
            CKD(cm->drv->wait64(cs, CUdeviceptr(mine + w), want, CU_STREAM_WAIT_VALUE_GEQ));
          }
          CK(cudaMemcpyAsync(mine, cm->flags(cm->rank) + FICCO_FLAG_CONST_ZERO, 8 * size_t(nwords),
                             cudaMemcpyDeviceToDevice, cs));
          break;
        }
        case FICCO_OP_RECORD:
          if (op.value >= FICCO_MAX_EVENTS) return fail(FICCO_EINVAL, "event slot out of range");
          CK(cudaEventRecord(cm->ev_pool[op.value], cs));
          break;
        case FICCO_OP_STREAM_WAIT:
          if (op.value >= FICCO_MAX_EVENTS) return fail(FICCO_EINVAL, "event slot out of range");
          CK(cudaStreamWaitEvent(cs, cm->ev_pool[op.value], 0));
          break;
        case FICCO_OP_REDUCE_MC: {
          uint8_t *src, *dst;
          int r = resolve(cm, parity, op.src_buf, -1, op.src_off, op.src_par, a, b, c, &src);
          if (r) return r;
          if ((r = resolve(cm, parity, op.dst_buf, op.dst_peer, op.dst_off, op.dst_par, a, b, c, &dst))) return r;
          const int64_t rows = op.height <= 1 ? 1 : op.height;
          const int64_t sp = rows > 1 ? op.src_pitch : op.width, dp = rows > 1 ? op.dst_pitch : op.width;
          const int64_t vecs = rows * (op.width / 16);
          const int grid = int(std::min<int64_t>(std::max<int64_t>(1, (vecs + 255) / 256), 4 * cm->sms));
          ficco::mc_reduce_kernel<<<grid, 256, 0, cs>>>(src, dst, rows, op.width, sp, dp);
          CK(cudaGetLastError());
          if (is_user(op.dst_buf)) {  // remember the node: later runs re-point it at the caller's output
            cudaStreamCaptureStatus st;
            CK(cudaStreamIsCapturing(cs, &st));
            if (st == cudaStreamCaptureStatusActive) {
              const cudaGraphNode_t* deps = nullptr;
              size_t nd = 0;
              CK(cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &deps, &nd));
              if (nd != 1) return fail(FICCO_ECUDA, "graph capture: reduce node not found");
              p->captured_reduces.push_back({deps[0], int(&op - p->ops.data())});
            }
          }
          break;
        }
        default: return fail(FICCO_EINVAL, "bad copy opcode " + std::to_string(op.op));
      }
    }
    for (int i = 0; i < p->n_streams; ++i) {
      CK(cudaEventRecord(cm->ev_join[i], cm->copy[i]));
      CK(cudaStreamWaitEvent(s, cm->ev_join[i], 0));
    }
  }
  CK(cudaEventRecord(cm->ev_join[FICCO_MAX_STREAMS - 1], side));
  CK(cudaStreamWaitEvent(s, cm->ev_join[FICCO_MAX_STREAMS - 1], 0));
  if (serialize) {
    int r = launch(p, parity, a, b, c, s);
    if (r) return r;
  }
  return 0;
}

int make_params(ficco_plan* p, uint32_t parity, const void* a, const void* b, void* c, ficco::TileParams* prm,
                int* grid) {
  ficco_comm* cm = p->comm;
  const ficco_plan_desc& d = p->desc;
  int r;
  memset(prm, 0, sizeof(*prm));
  uint8_t *pa, *pb;
  if ((r = resolve(cm, parity, d.a.buf, -1, d.a.off, d.a.par, a, b, c, &pa))) return r;
  if ((r = resolve(cm, parity, d.b.buf, -1, d.b.off, d.b.par, a, b, c, &pb))) return r;
  if ((r = encode_bf16_2d(cm->drv, &prm->tmap_a, pa, d.a.rows, d.k, d.a.ld, ficco::BM))) return r;
  {
    const void* fn;
    int smem, b_rows, stages;
    if ((r = kernel_for(p->tile_n, p->cta_group, p->epi_bufs, &fn, &smem, &b_rows, &stages))) return r;
    if ((r = encode_bf16_2d(cm->drv, &prm->tmap_b, pb, d.b.rows, d.k, d.b.ld, b_rows))) return r;
    // B-resident mode for short-K programs without REDUCE tiles (their identity-MMA boxes use the B slots):
    // consecutive tiles of a CTA that share B rows stream only A (FICCO_B_RESIDENT=0/1 overrides)
    const char* env = getenv("FICCO_B_RESIDENT");
    const int kbs = int((d.k + ficco::BK - 1) / ficco::BK);
    const bool can = kbs <= stages && p->role != ROLE_REDUCE_SCATTER;
    prm->b_resident = can && (env ? env[0] == '1' : kbs <= 4) ? 1 : 0;
    prm->tmap_a2 = prm->tmap_a;
    prm->tmap_b2 = prm->tmap_b;
    if (d.a2.buf != FICCO_BUF_NONE) {
      uint8_t* p2;
      if ((r = resolve(cm, parity, d.a2.buf, -1, d.a2.off, d.a2.par, a, b, c, &p2))) return r;
      if ((r = encode_bf16_2d(cm->drv, &prm->tmap_a2, p2, d.a2.rows, d.k, d.a2.ld, ficco::BM))) return r;
    }
    if (d.b2.buf != FICCO_BUF_NONE) {
      uint8_t* p2;
      if ((r = resolve(cm, parity, d.b2.buf, -1, d.b2.off, d.b2.par, a, b, c, &p2))) return r;
      if ((r = encode_bf16_2d(cm->drv, &prm->tmap_b2, p2, d.b2.rows, d.k, d.b2.ld, b_rows))) return r;
    }
  }
  uint8_t* po = nullptr;
  if (d.c.buf != FICCO_BUF_NONE && (r = resolve(cm, parity, d.c.buf, -1, d.c.off, d.c.par, a, b, c, &po))) return r;
  uint8_t* pp = nullptr;
  if (d.part.buf != FICCO_BUF_NONE &&
      (r = resolve(cm, parity, d.part.buf, -1, d.part.off, d.part.par, a, b, c, &pp)))
    return r;
  if (po && d.c.rows > 0) {
    if ((r = encode_store_map(cm->drv, &prm->tmap_out, po, d.c.rows, d.c.ld, d.c.ld, 64))) return r;
    if ((r = encode_store_map(cm->drv, &prm->tmap_out32, po, d.c.rows, d.c.ld, d.c.ld, 32))) return r;
    prm->has_out_map = 1;
  }
  if (pp && d.part.rows > 0) {
    if ((r = encode_store_map(cm->drv, &prm->tmap_part, pp, d.part.rows, d.part.ld, d.part.ld, 64))) return r;
    if ((r = encode_store_map(cm->drv, &prm->tmap_part32, pp, d.part.rows, d.part.ld, d.part.ld, 32))) return r;
    prm->has_part_map = 1;
  }
  prm->tiles = p->d_tiles;
  prm->num_tiles = p->n_tiles;
  prm->num_kb = int((d.k + ficco::BK - 1) / ficco::BK);
  prm->out = reinterpret_cast<__nv_bfloat16*>(po);
  prm->part = reinterpret_cast<__nv_bfloat16*>(pp);
  prm->ld_out = d.c.ld;
  prm->ld_part = d.part.ld;
  prm->n_recv = d.n_recv;
  for (int j = 0; j < d.n_recv; ++j) {
    uint8_t* pr;
    if ((r = resolve(cm, parity, d.recv.buf, -1, d.recv.off + j * d.recv_slot, d.recv.par, a, b, c, &pr))) return r;
    prm->recv[j] = reinterpret_cast<const __nv_bfloat16*>(pr);
  }
  prm->ld_recv = d.recv.ld;
  prm->rs_flag0 = d.rs_flag0;
  {
    // identity-MMA reduction: the receive slots must tile one [n_recv * rows, N] matrix
    const char* hint = getenv("FICCO_PART_HINT");
    prm->part_hint = hint ? atoi(hint) : 0;
    const char* env = getenv("FICCO_RS_MMA");
    const int64_t pitch = d.recv.ld * 2;
    if (d.n_recv > 0 && !(env && env[0] == '0') && pitch > 0 && d.recv_slot % pitch == 0) {
      uint8_t* pr0;
      if ((r = resolve(cm, parity, d.recv.buf, -1, d.recv.off, d.recv.par, a, b, c, &pr0))) return r;
      prm->recv_rows = int(d.recv_slot / pitch);
      if ((r = encode_bf16_2d(cm->drv, &prm->tmap_recv, pr0, int64_t(d.n_recv) * prm->recv_rows, d.recv.ld,
                              d.recv.ld, ficco::BM)))
        return r;
      if ((r = encode_bf16_2d(cm->drv, &prm->tmap_ident, cm->ws[cm->rank] + FICCO_WS_IDENTITY_OFF, 64, 64, 64,
                              64 / p->cta_group)))
        return r;
      const char* alias = getenv("FICCO_RS_ALIAS");  // timing experiments only: every peer reads slot 0
      if (alias && alias[0] == '1') prm->recv_rows = 0;
      prm->reduce_mma = env && env[0] == '2' ? 2 : 1;  // 2: loads without the identity MMAs (timing only)
    }
  }
  if (p->has_remote) {
    // this rank's receive slot on every owner q (symmetric workspaces: same offsets everywhere)
    for (int q = 0; q < cm->world; ++q) {
      if (q == cm->rank) continue;
      const int slot = cm->rank < q ? cm->rank : cm->rank - 1;
      uint8_t* base;
      if ((r = resolve(cm, parity, d.recv.buf, q, d.recv.off + slot * d.recv_slot, d.recv.par, a, b, c, &base)))
        return r;
      if ((r = encode_store_map(cm->drv, &prm->tmap_rem[q], base, d.recv.rows, d.recv.ld, d.recv.ld, 64))) return r;
      if ((r = encode_store_map(cm->drv, &prm->tmap_rem32[q], base, d.recv.rows, d.recv.ld, d.recv.ld, 32)))
        return r;
      prm->rem[q] = reinterpret_cast<__nv_bfloat16*>(base);
      prm->rem_flags[q] = cm->block(q, parity);
    }
    prm->ld_rem = d.recv.ld;
    prm->has_rem_map = 1;
  }
  prm->go_flag = d.go_flag;
  prm->go_all = d.part.buf == FICCO_BUF_MC ? 1 : 0;  // nvls: the multicast-bound partials are read by peers
  prm->rs_target = d.rs_target > 0 ? uint32_t(d.rs_target) : 1u;
  prm->flags = cm->block(cm->rank, parity);
  prm->counters = cm->block(cm->rank, parity) + FICCO_FLAG_COUNTERS;
  prm->abort_word = cm->flags(cm->rank) + FICCO_FLAG_ABORT;
  prm->abort_host = cm->dev_host_abort;
  prm->epoch = 1u;  // one-shot flags: wait for != 0
  {
    // a flag wait longer than this is a protocol failure (FICCO_ETIMEOUT -> DeadlockError); ops of
    // many seconds (the reference's largest grid shapes) may need more via FICCO_FLAG_TIMEOUT_S
    const char* t = getenv("FICCO_FLAG_TIMEOUT_S");
    const double sec = t ? atof(t) : 30.0;
    prm->timeout_ns = static_cast<unsigned long long>((sec > 0 ? sec : 30.0) * 1e9);
  }
  prm->alpha = d.alpha;
  prm->a_evict_last = (d.hints & FICCO_HINT_A_EVICT_LAST) != 0;
  {
    // Output stores: evict_first (keeps operands L2-resident). The epilogue-only probe writes HBM faster
    // with plain stores (tools/epi_probe.cu), but in the tile kernel with the fast epilogue path and
    // resident B, evict_first measured 2-3 % faster on C4 (tools/out_hint_ab.py). FICCO_OUT_HINT=none
    // selects plain stores.
    const char* env = getenv("FICCO_OUT_HINT");
    prm->out_plain = env && env[0] == 'n' ? 1 : 0;
    const char* fast = getenv("FICCO_EPI_FAST");
    prm->epi_fast = fast && fast[0] == '0' ? 0 : 1;
    const char* x64 = getenv("FICCO_EPI_X64");
    prm->epi_x64 = x64 && x64[0] == '1' ? 1 : 0;
  }
  prm->b_evict_first = (d.hints & FICCO_HINT_B_EVICT_FIRST) != 0;
  {
    // FICCO_B_HINT=last|first|normal overrides the plan's B (weight) L2 policy (A/B experiments)
    const char* env = getenv("FICCO_B_HINT");
    if (env && env[0]) prm->b_evict_first = env[0] == 'f' ? 1 : env[0] == 'n' ? 2 : 0;
  }
  prm->trace = p->trace;
  int g = d.grid > 0 ? d.grid : cm->sms;
  if (g > p->n_tiles) g = p->n_tiles;
  if (p->cta_group == 2) g &= ~1;  // whole clusters
  *grid = g;
  return 0;
}

// The launch-time knobs make_params reads (experiments toggle them between calls).
std::string knob_fingerprint() {
  static const char* const names[] = {"FICCO_B_RESIDENT", "FICCO_PART_HINT", "FICCO_RS_MMA", "FICCO_RS_ALIAS",
                                      "FICCO_FLAG_TIMEOUT_S", "FICCO_OUT_HINT", "FICCO_EPI_FAST", "FICCO_B_HINT",
                                      "FICCO_EPI_X64"};
  std::string f;
  for (const char* n : names) {
    const char* v = getenv(n);
    f += v ? v : "\x01";
    f += '\x02';
  }
  return f;
}

int launch_tiles(ficco_plan* p, uint32_t parity, const void* a, const void* b, void* c, cudaStream_t s) {
  if (p->n_tiles == 0) return 0;
  int r = configure_kernels(p->comm->device);
  if (r) return r;
  int grid, smem, b_rows;
  const void* fn;
  if ((r = kernel_for(p->tile_n, p->cta_group, p->epi_bufs, &fn, &smem, &b_rows))) return r;
  ficco_plan::ParamCache& pc = p->pcache[parity & 1u];
  std::string knobs = knob_fingerprint();
  if (!(pc.valid && pc.a == a && pc.b == b && pc.c == c && pc.trace == p->trace && pc.knobs == knobs)) {
    pc.valid = false;
    if ((r = make_params(p, parity, a, b, c, &pc.prm, &pc.grid))) return r;
    pc.a = a, pc.b = b, pc.c = c, pc.trace = p->trace, pc.knobs = std::move(knobs), pc.valid = true;
  }
  ficco::TileParams& prm = pc.prm;
  grid = pc.grid;
  void* args[] = {&prm};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ficco::NUM_THREADS);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(p->cta_group);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelExC(&cfg, fn, args));
  cudaStreamCaptureStatus st;
  CK(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive) {  // remember the kernel node so later runs can re-point it
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd));
    p->captured_kernel = nd == 1 ? deps[0] : nullptr;
  }
  return 0;
}

int build_graph(ficco_plan* p, uint32_t parity, const void* a, const void* b, void* c, cudaStream_t s) {
  GraphInst& gi = p->graph[parity];
  cudaStream_t cap;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  p->captured_kernel = nullptr;
  p->captured_copies.clear();
  p->captured_reduces.clear();
  int r = enqueue_run(p, parity, a, b, c, cap, true, p->kernel_in_graph, launch_tiles);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(cap, &graph);
  cudaStreamDestroy(cap);
  if (r) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  if (e != cudaSuccess) return fail(FICCO_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  gi.kernel = p->captured_kernel;
  gi.user_copies = p->captured_copies;
  gi.user_reduces = p->captured_reduces;
  p->captured_kernel = nullptr;
  p->captured_copies.clear();
  p->captured_reduces.clear();
  if (p->kernel_in_graph && p->n_tiles > 0 && !gi.kernel) {
    cudaGraphDestroy(graph);
    return fail(FICCO_ECUDA, "graph capture: kernel node not found");
  }
  if (gi.exec) cudaGraphExecDestroy(gi.exec);
  if (gi.graph) cudaGraphDestroy(gi.graph);
  gi.exec = nullptr;
  gi.graph = graph;
  e = cudaGraphInstantiate(&gi.exec, graph, 0);
  if (e != cudaSuccess) return fail(FICCO_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  gi.a = a;
  gi.b = b;
  gi.c = c;
  return 0;
}

int repoint_graph(ficco_plan* p, uint32_t parity, const void* a, const void* b, void* c) {
  GraphInst& gi = p->graph[parity];
  if (gi.kernel) {
    ficco::TileParams prm;
    int grid;
    int r = make_params(p, parity, a, b, c, &prm, &grid);
    if (r) return r;
    void* args[] = {&prm};
    const void* fn;
    int smem, b_rows;
    if ((r = kernel_for(p->tile_n, p->cta_group, p->epi_bufs, &fn, &smem, &b_rows))) return r;
    cudaKernelNodeParams kp{};
    kp.func = const_cast<void*>(fn);
    kp.gridDim = dim3(grid);
    kp.blockDim = dim3(ficco::NUM_THREADS);
    kp.sharedMemBytes = size_t(smem);
    kp.kernelParams = args;
    CK(cudaGraphExecKernelNodeSetParams(gi.exec, gi.kernel, &kp));
  }
  for (auto& nc : gi.user_copies) {
    const ficco_copy_op& op = p->ops[nc.second];
    uint8_t *src, *dst;
    int r = resolve(p->comm, parity, op.src_buf, op.peer, op.src_off, op.src_par, a, b, c, &src);
    if (r) return r;
    if ((r = resolve(p->comm, parity, op.dst_buf, op.dst_peer, op.dst_off, op.dst_par, a, b, c, &dst))) return r;
    CK(cudaGraphExecMemcpyNodeSetParams1D(gi.exec, nc.first, dst, src, size_t(op.width), cudaMemcpyDefault));
  }
  for (auto& nr : gi.user_reduces) {
    const ficco_copy_op& op = p->ops[nr.second];
    uint8_t *src, *dst;
    int r = resolve(p->comm, parity, op.src_buf, -1, op.src_off, op.src_par, a, b, c, &src);
    if (r) return r;
    if ((r = resolve(p->comm, parity, op.dst_buf, op.dst_peer, op.dst_off, op.dst_par, a, b, c, &dst))) return r;
    cudaKernelNodeParams kp{};
    CK(cudaGraphKernelNodeGetParams(nr.first, &kp));
    const int64_t rows = op.height <= 1 ? 1 : op.height;
    int64_t width = op.width, sp = rows > 1 ? op.src_pitch : op.width, dp = rows > 1 ? op.dst_pitch : op.width;
    const uint8_t* s8 = src;
    uint8_t* d8 = dst;
    int64_t rows_v = rows;
    void* args[] = {&s8, &d8, &rows_v, &width, &sp, &dp};
    kp.kernelParams = args;
    kp.extra = nullptr;
    CK(cudaGraphExecKernelNodeSetParams(gi.exec, nr.first, &kp));
  }
  gi.a = a;
  gi.b = b;
  gi.c = c;
  return 0;
}

// A run of this communicator timed out on a readiness flag (the kernel drained without its
// inputs): its flag words and workspaces are in an unknown state, so it refuses further runs.
bool poisoned(const ficco_comm* c) { return c->host_abort && *reinterpret_cast<volatile uint32_t*>(c->host_abort); }
int poisoned_error() {
  return fail(FICCO_ETIMEOUT,
              "communicator poisoned: an earlier run timed out waiting for a readiness flag; destroy the "
              "communicator (FiccoGroup.close) and create a new one");
}

}  // namespace

extern "C" {

int ficco_abi_version(void) { return FICCO_ABI_VERSION; }
const char* ficco_last_error(void) { return g_err.c_str(); }

int ficco_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return 0;
}

int ficco_ws_alloc(size_t bytes, void** out) {
  if (!out || bytes < FICCO_WS_DATA_OFFSET) return fail(FICCO_EINVAL, "workspace smaller than flag area");
  void* p = nullptr;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMemset(p, 0, FICCO_WS_DATA_OFFSET));
  const uint32_t one = 0x01010101u;
  CK(cudaMemcpy(reinterpret_cast<uint32_t*>(p) + FICCO_FLAG_CONST_ONE, &one, 4, cudaMemcpyHostToDevice));
  {
    uint16_t ident[64 * 64] = {};
    for (int i = 0; i < 64; ++i) ident[i * 64 + i] = 0x3F80;  // bf16 1.0
    CK(cudaMemcpy(reinterpret_cast<uint8_t*>(p) + FICCO_WS_IDENTITY_OFF, ident, sizeof(ident),
                  cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  *out = p;
  return 0;
}

int ficco_ws_free(void* ptr) {
  CK(cudaFree(ptr));
  return 0;
}

int ficco_ipc_handle_size(void) { return int(sizeof(cudaIpcMemHandle_t)); }

int ficco_ipc_get_handle(void* ptr, void* out_handle) {
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ptr));
  memcpy(out_handle, &h, sizeof(h));
  return 0;
}

int ficco_ipc_open(const void* handle, void** out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int ficco_ipc_close(void* ptr) {
  CK(cudaIpcCloseMemHandle(ptr));
  return 0;
}

int ficco_comm_create(int rank, int world, void* const* ws, size_t ws_bytes, int virtual_peers, ficco_comm_t** out) {
  if (!out || !ws || world < 1 || rank < 0 || rank >= world) return fail(FICCO_EINVAL, "bad comm arguments");
  if (ws_bytes < FICCO_WS_DATA_OFFSET) return fail(FICCO_EINVAL, "workspace smaller than flag area");
  Driver* drv;
  int r = get_driver(&drv);
  if (r) return r;
  int dev;
  CK(cudaGetDevice(&dev));
  int sms, major;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) return fail(FICCO_ENODEV, "libficco_b200 needs an sm_100 (B200) device");
  auto* c = new ficco_comm();
  c->rank = rank;
  c->world = world;
  c->device = dev;
  c->sms = sms;
  c->virt = virtual_peers != 0;
  c->ws_bytes = ws_bytes;
  c->drv = drv;
  for (int i = 0; i < world; ++i) c->ws.push_back(reinterpret_cast<uint8_t*>(ws[i]));
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&c->host_abort), 4, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *c->host_abort = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dev_host_abort), c->host_abort, 0);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  for (int i = 0; i < FICCO_MAX_STREAMS && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&c->copy[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming);
  }
  for (int i = 0; i < FICCO_MAX_EVENTS && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&c->ev_pool[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ficco_comm_destroy(c);
    return fail(FICCO_ECUDA, std::string("comm stream/event creation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return 0;
}

int ficco_comm_destroy(ficco_comm_t* c) {
  if (!c) return 0;
  for (int i = 0; i < FICCO_MAX_STREAMS; ++i) {
    if (c->copy[i]) {
      cudaStreamSynchronize(c->copy[i]);
      cudaStreamDestroy(c->copy[i]);
    }
    if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
  }
  for (int i = 0; i < FICCO_MAX_EVENTS; ++i)
    if (c->ev_pool[i]) cudaEventDestroy(c->ev_pool[i]);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->host_abort) cudaFreeHost(c->host_abort);
  delete c;
  return 0;
}

int ficco_comm_epoch(ficco_comm_t* c, uint32_t* runs) {
  if (!c || !runs) return fail(FICCO_EINVAL, "null argument");
  *runs = c->runs;
  return 0;
}

int ficco_comm_check(ficco_comm_t* c, void* stream) {
  if (!c) return fail(FICCO_EINVAL, "null comm");
  CK(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  for (int i = 0; i < FICCO_MAX_STREAMS; ++i) CK(cudaStreamSynchronize(c->copy[i]));
  uint32_t abort_word = 0;
  CK(cudaMemcpy(&abort_word, c->flags(c->rank) + FICCO_FLAG_ABORT, 4, cudaMemcpyDeviceToHost));
  if (abort_word || *reinterpret_cast<volatile uint32_t*>(c->host_abort)) {
    std::string where;
    if (abort_word & 0x80000000u) {  // the word's address (low 31 bits) -> flag block / index, if it is local
      const uint32_t base = uint32_t(reinterpret_cast<uintptr_t>(c->flags(c->rank))) & 0x7fffffffu;
      const int64_t off = (int64_t(abort_word & 0x7fffffffu) - int64_t(base)) / 4;
      if (off >= 0 && off < FICCO_WS_FLAG_WORDS)
        where = " (flag block " + std::to_string(off / FICCO_FLAG_BLOCK) + ", word " +
                std::to_string(off % FICCO_FLAG_BLOCK) + ")";
    }
    return fail(FICCO_ETIMEOUT, "tile kernel timed out waiting for a readiness flag" + where);
  }
  return 0;
}

int ficco_comm_set_flags(ficco_comm_t* c, int first, int count, uint32_t value, void* stream) {
  if (!c || first < 0 || count < 0 || first + count > FICCO_WS_FLAG_WORDS) return fail(FICCO_EINVAL, "bad flag range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < count; ++i) CKD(c->drv->write32(s, CUdeviceptr(c->flags(c->rank) + first + i), value, 0));
  return 0;
}

int ficco_plan_create(ficco_comm_t* c, const ficco_plan_desc* d, ficco_plan_t** out) {
  if (!c || !d || !out) return fail(FICCO_EINVAL, "null argument");
  if (d->n_tiles < 0 || d->n_ops < 0) return fail(FICCO_EINVAL, "negative program length");
  if (d->n_tiles > 0 && (d->k <= 0 || d->k % 8 != 0)) return fail(FICCO_EINVAL, "K must be a positive multiple of 8");
  if (d->n_recv < 0 || d->n_recv > ficco::MAX_RECV) return fail(FICCO_EINVAL, "too many receive slots");
  if (d->n_counters < 0 || FICCO_FLAG_COUNTERS + d->n_counters > FICCO_FLAG_BLOCK)
    return fail(FICCO_EINVAL, "too many counters");
  const int tile_n = d->tile_n > 0 ? d->tile_n : 256;
  const int cta_group = d->cta_group > 0 ? d->cta_group : 1;
  {
    const void* fn;
    int smem, b_rows;
    int r = kernel_for(tile_n, cta_group, epi_bufs_for(d->k), &fn, &smem, &b_rows);
    if (r) return r;
    if (cta_group == 2 && d->n_tiles % 2) return fail(FICCO_EINVAL, "cta_group 2 needs an even tile list (pairs)");
  }
  bool has_remote = false;
  for (int i = 0; i < d->n_tiles; ++i) {
    const ficco_tile& t = d->tiles[i];
    if (t.rows < 0 || t.rows > ficco::BM || (t.rows == 0 && cta_group == 1) || t.cols < 32 || t.cols > tile_n ||
        t.cols % 32)
      return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": rows/cols out of range");
    if (t.mode < FICCO_EPI_STORE || t.mode > FICCO_EPI_STORE_REMOTE)
      return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": bad epilogue mode");
    if (t.mode == FICCO_EPI_STORE_REMOTE) {
      if (t.chunk < 0 || t.chunk >= c->world || t.chunk == c->rank || c->world > ficco::MAX_PEERS)
        return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": STORE_REMOTE owner rank out of range");
      if (t.recv_row < FICCO_FLAG_RUN_LOCAL || t.recv_row >= FICCO_FLAG_BLOCK)
        return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": STORE_REMOTE flag out of the run-local block");
      has_remote = true;
    }
    if (t.flag >= 0) {
      int top = 15;
      while (top > 0 && !(t.fmask & (1u << top))) --top;
      const int last = t.flag + top + (t.kseg ? (int((d->k + 63) / 64) / t.kseg) * t.kstride : 0);
      if (t.fmask == 0 || last >= FICCO_FLAG_BLOCK || t.kseg < 0)
        return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": flag range out of the flag block");
    }
    if ((t.a_src && d->a2.buf == FICCO_BUF_NONE) || (t.b_src && d->b2.buf == FICCO_BUF_NONE))
      return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": alternate operand not provided");
  }
  int n_streams = 0;
  bool user = false;
  for (int i = 0; i < d->n_ops; ++i) {
    const ficco_copy_op& op = d->ops[i];
    if (op.stream < 0 || op.stream >= FICCO_MAX_STREAMS - 1) return fail(FICCO_EINVAL, "op stream out of range");
    if (op.op < FICCO_OP_COPY || op.op > FICCO_OP_REDUCE_MC) return fail(FICCO_EINVAL, "bad copy opcode");
    if (op.op == FICCO_OP_REDUCE_MC && (op.src_buf != FICCO_BUF_MCV || op.width % 16 ||
                                        (op.height > 1 && (op.src_pitch % 16 || op.dst_pitch % 16))))
      return fail(FICCO_EINVAL, "REDUCE_MC reads the multicast view in 16-byte vectors");
    if ((op.src_buf == FICCO_BUF_MC || op.src_buf == FICCO_BUF_MCV || op.dst_buf == FICCO_BUF_MC ||
         op.dst_buf == FICCO_BUF_MCV) && !c->mc_va)
      return fail(FICCO_ENODEV, "the plan uses the multicast (NVLS) workspace but the communicator has none "
                                "(ficco_comm_set_multicast)");
    if ((op.op == FICCO_OP_SIGNAL || op.op == FICCO_OP_NOTIFY || op.op == FICCO_OP_WAIT ||
         op.op == FICCO_OP_BARRIER) && (op.flag < 0 || op.flag + 4 > FICCO_FLAG_BLOCK))
      return fail(FICCO_EINVAL, "op flag index out of range");
    if (op.op == FICCO_OP_SIGNAL && op.value > 1 && op.flag + int64_t(op.value) > FICCO_FLAG_BLOCK)
      return fail(FICCO_EINVAL, "signal run out of the flag block");
    if (op.op == FICCO_OP_COPY && (is_user(op.src_buf) || is_user(op.dst_buf))) user = true;
    if (op.stream + 1 > n_streams) n_streams = op.stream + 1;
  }
  if (has_remote && (d->recv.rows <= 0 || d->recv.ld <= 0))
    return fail(FICCO_EINVAL, "STORE_REMOTE tiles need the receive-slot geometry (recv)");
  if (d->part.buf == FICCO_BUF_MC && (!c->mc_uc || d->part.off + d->part.rows * d->part.ld * 2 >
                                                       int64_t(c->mc_bytes)))
    return fail(FICCO_ENODEV, "partials in the multicast (NVLS) workspace need ficco_comm_set_multicast with "
                              "enough bytes");
  auto* p = new ficco_plan();
  p->comm = c;
  p->desc = *d;
  p->ops.assign(d->ops, d->ops + d->n_ops);
  for (const ficco_copy_op& op : p->ops) p->counter_waits |= op.op == FICCO_OP_WAIT_COUNTER;
  p->desc.ops = nullptr;
  p->desc.tiles = nullptr;
  p->n_tiles = d->n_tiles;
  p->tile_n = tile_n;
  p->cta_group = cta_group;
  p->epi_bufs = epi_bufs_for(d->k);
  p->has_remote = has_remote;
  p->role = plan_role(*d);
  {
    const char* env = getenv("FICCO_KERNEL_IN_GRAPH");
    p->kernel_in_graph = env && env[0] == '1';
  }
  if (cta_group == 2 && p->desc.grid % 2) p->desc.grid = p->desc.grid > 1 ? p->desc.grid - 1 : 2;  // whole pairs
  p->n_streams = n_streams;
  p->user_copies = user;
  if (d->n_tiles > 0) {
    size_t bytes = sizeof(ficco_tile) * size_t(d->n_tiles);
    cudaError_t e = cudaMalloc(&p->d_tiles, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_tiles, d->tiles, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(p->d_tiles);
      delete p;
      return fail(FICCO_ECUDA, std::string("tile upload: ") + cudaGetErrorString(e));
    }
  }
  *out = p;
  return 0;
}

int ficco_plan_destroy(ficco_plan_t* p) {
  if (!p) return 0;
  for (auto& g : p->graph) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  if (p->d_tiles) cudaFree(p->d_tiles);
  delete p;
  return 0;
}

int ficco_plan_set_trace(ficco_plan_t* p, void* buf) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  p->trace = reinterpret_cast<unsigned long long*>(buf);
  for (auto& g : p->graph) {  // rebuild on next run with the new kernel parameters
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g = GraphInst{};
  }
  return 0;
}

int ficco_plan_set_kernel_event(ficco_plan_t* p, void* event) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  if (p->kernel_in_graph && event) return fail(FICCO_EINVAL, "kernel events need the direct kernel launch mode");
  p->kernel_event = reinterpret_cast<cudaEvent_t>(event);
  return 0;
}

int ficco_plan_info(ficco_plan_t* p, int* n_tiles, int* grid, int* n_streams) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  int g = p->desc.grid > 0 ? p->desc.grid : p->comm->sms;
  if (g > p->n_tiles) g = p->n_tiles;
  if (n_tiles) *n_tiles = p->n_tiles;
  if (grid) *grid = g;
  if (n_streams) *n_streams = p->n_streams;
  return 0;
}

int ficco_plan_run_parts(ficco_plan_t* p, const void* a, const void* b, void* c, void* stream, int run_copies,
                         int run_tiles) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  if (poisoned(p->comm)) return poisoned_error();
  p->concurrent = run_tiles != 2;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t parity = p->comm->runs & 1u;
  p->comm->runs += 1;
  return enqueue_run(p, parity, a, b, c, s, run_copies != 0, run_tiles != 0, launch_tiles);
}

int ficco_plan_run(ficco_plan_t* p, const void* a, const void* b, void* c, void* stream) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  if (poisoned(p->comm)) return poisoned_error();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t parity = p->comm->runs & 1u;
  GraphInst& gi = p->graph[parity];
  int r;
  if (!gi.exec) {
    if ((r = build_graph(p, parity, a, b, c, s))) return r;
  } else if (gi.a != a || gi.b != b || gi.c != c) {
    if ((r = repoint_graph(p, parity, a, b, c))) return r;  // user-buffer copy nodes (+ kernel node)
  }
  p->comm->runs += 1;
  if (p->kernel_in_graph) {
    CK(cudaGraphLaunch(gi.exec, s));
    return 0;
  }
  // Launch order. A copy program that waits on tile counters (GEMM -> RS with copy-engine pushes, NVLS)
  // goes after the kernel: the kernel is then dispatched before any of the graph's stream-wait nodes
  // exists, so a blocked wait can never hold back the kernel that satisfies it. Every other copy
  // program waits only on peers' copy programs, so it goes first and its copies start earlier
  // (C2 hetero_unfused_1d -1.6 / -2.1 %, others unchanged: profiles/r02_experiments/graph_first_ab.json).
  // FICCO_GRAPH_FIRST=0 restores kernel-first for every plan.
  ficco_comm* cm = p->comm;
  cudaStream_t gs = cm->copy[FICCO_MAX_STREAMS - 1];  // graph launch stream (idle between runs)
  const char* gf = getenv("FICCO_GRAPH_FIRST");
  const bool graph_first = !(gf && gf[0] == '0') && !p->counter_waits;
  CK(cudaEventRecord(cm->ev_fork, s));
  if (graph_first) {
    CK(cudaStreamWaitEvent(gs, cm->ev_fork, 0));
    CK(cudaGraphLaunch(gi.exec, gs));
  }
  if ((r = launch_tiles(p, parity, a, b, c, s))) return r;
  if (p->kernel_event) CK(cudaEventRecord(p->kernel_event, s));  // completes with the tile kernel
  if (!graph_first) {
    CK(cudaStreamWaitEvent(gs, cm->ev_fork, 0));
    CK(cudaGraphLaunch(gi.exec, gs));
  }
  CK(cudaEventRecord(cm->ev_join[0], gs));
  CK(cudaStreamWaitEvent(s, cm->ev_join[0], 0));
  return 0;
}

namespace {
int run_as(ficco_plan_t* p, int role, const char* op, const void* a, const void* b, void* c, void* stream) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  if (p->role != role) return fail(FICCO_EINVAL, std::string(op) + ": the plan was not lowered for this op");
  return ficco_plan_run(p, a, b, c, stream);
}
}  // namespace

int ficco_ag_gemm(ficco_plan_t* plan, const void* a_shard, const void* w, void* c, void* stream) {
  return run_as(plan, ROLE_GATHER_A, "ficco_ag_gemm", a_shard, w, c, stream);
}
int ficco_a2a_gemm(ficco_plan_t* plan, const void* a_send, const void* w, void* c, void* stream) {
  return run_as(plan, ROLE_GATHER_A, "ficco_a2a_gemm", a_send, w, c, stream);
}
int ficco_gemm_rs(ficco_plan_t* plan, const void* a, const void* w, void* c_shard, void* stream) {
  return run_as(plan, ROLE_REDUCE_SCATTER, "ficco_gemm_rs", a, w, c_shard, stream);
}
int ficco_cp_qk(ficco_plan_t* plan, const void* q, const void* k_shard, void* scores, void* stream) {
  return run_as(plan, ROLE_GATHER_B, "ficco_cp_qk", q, k_shard, scores, stream);
}

int ficco_timestamp(void* dst, void* stream) {
  ficco::stamp_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(reinterpret_cast<unsigned long long*>(dst));
  CK(cudaGetLastError());
  return 0;
}

int ficco_watch_words(const void* words, int n, uint32_t want, void* out, int64_t timeout_ns, void* stream) {
  if (n <= 0 || n > 4096) return fail(FICCO_EINVAL, "watch: 1..4096 words");
  ficco::watch_kernel<<<1, n < 1024 ? n : 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint32_t*>(words), n, want, reinterpret_cast<unsigned long long*>(out), timeout_ns);
  CK(cudaGetLastError());
  return 0;
}

int ficco_occupy_sms(int64_t ns, void* stream) {
  int dev, sms, smem;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  CK(cudaFuncSetAttribute(ficco::occupy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  ficco::occupy_kernel<<<sms, 1024, smem, reinterpret_cast<cudaStream_t>(stream)>>>(ns);
  CK(cudaGetLastError());
  return 0;
}

int ficco_copy_batch(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t count, void* stream) {
  // one stream-ordered copy per entry (the driver's batched-copy entry point is not used: it faulted
  // the GPU on this pool)
  for (size_t i = 0; i < count; ++i)
    CK(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

int ficco_gemm_bf16_cfg(const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k, float alpha,
                        int grid, int tile_n, int cta_group, void* stream) {
  // Plain C = alpha * A @ B^T through the same tile kernel (no flags), cached per shape/config.
  if (m <= 0 || n <= 0 || k <= 0 || n % 32 || k % 8) return fail(FICCO_EINVAL, "gemm: need N%32==0, K%8==0");
  if (cta_group == 0) cta_group = 2;
  if (cta_group != 1 && cta_group != 2) return fail(FICCO_EINVAL, "cta_group must be 1 or 2");
  static std::mutex mu;
  // keyed on the full shape: the tile width, raster grouping and L2 hints all depend on (m, n, k)
  static std::map<std::tuple<int64_t, int64_t, int64_t, int, int, int, int, int64_t>,
                  std::pair<ficco_comm*, ficco_plan*>>
      cache;
  std::lock_guard<std::mutex> lock(mu);
  int dev;
  CK(cudaGetDevice(&dev));
  const char* genv = getenv("FICCO_GEMM_GROUP_M");  // pair-blocks per raster group (A/B experiments)
  auto key = std::make_tuple(m, n, k, grid, dev, tile_n, cta_group, genv ? atoll(genv) : int64_t(-1));
  auto it = cache.find(key);
  if (it == cache.end()) {
    static std::map<int, void*> ws_by_dev;
    if (!ws_by_dev.count(dev)) {
      void* w;
      int r = ficco_ws_alloc(FICCO_WS_DATA_OFFSET, &w);
      if (r) return r;
      ws_by_dev[dev] = w;
    }
    ficco_comm* cm;
    void* w = ws_by_dev[dev];
    int r = ficco_comm_create(0, 1, &w, FICCO_WS_DATA_OFFSET, 1, &cm);
    if (r) return r;
    int tn = tile_n;
    if (tn == 0) {  // tile width minimising waves x (width + 512) (lowering.choose_tile_n: a tile's A slab
                    // streams through L2 -> SMEM whatever its width)
      double best = 1e30;
      const int widths[] = {256, 224, 192, 160, 128};
      const int units = cm->sms / cta_group;
      for (int wdt : widths) {
        const int64_t tiles_n = (n + wdt - 1) / wdt;
        const int64_t tiles_m = ((m + ficco::BM - 1) / ficco::BM + cta_group - 1) / cta_group;
        const int64_t waves = (tiles_n * tiles_m + units - 1) / units;
        const double cost = double(waves) * (wdt + 512);
        if (cost < best - 1e-9) {
          best = cost;
          tn = wdt;
        }
      }
    }
    std::vector<ficco_tile> tiles;
    const int64_t mstep = int64_t(ficco::BM) * cta_group;
    auto push = [&](int64_t i, int64_t j, bool pad) {
      for (int h = 0; h < cta_group; ++h) {
        const int64_t row = i + h * ficco::BM;
        ficco_tile t{};
        t.a_row = int32_t(row < m ? row : i);
        t.b_row = int32_t(j);
        t.c_row = int32_t(row);
        t.c_col = int32_t(j);
        t.rows = int16_t(pad || row >= m ? 0 : (m - row < ficco::BM ? m - row : ficco::BM));
        t.cols = int16_t(n - j < tn ? n - j : tn);
        t.flag = -1;
        t.fmask = 0;
        t.mode = FICCO_EPI_STORE;
        tiles.push_back(t);
      }
    };
    const int64_t slots = (grid > 0 ? grid : cm->sms) / cta_group;
    const int64_t ncb = (n + tn - 1) / tn;
    const char* benv = getenv("FICCO_B_RESIDENT");
    if (!genv && cta_group == 2 && k <= 256 && ncb >= slots && !(benv && benv[0] == '0')) {
      // short K (store-bound, b_resident): waves of `slots` column blocks listed row-block by row-block, so
      // CTA pair p (which takes pair-tiles p, p + slots, ...) keeps ONE column block of B in smem for all of
      // M and streams only A; a partial last wave is padded with load-only pair tiles to keep the mapping
      for (int64_t w0 = 0; w0 < ncb; w0 += slots)
        for (int64_t i = 0; i < m; i += mstep)
          for (int64_t u = w0; u < w0 + slots; ++u) push(i, (u < ncb ? u : w0) * tn, u >= ncb);
    } else {
      const int64_t group = genv ? std::max<int64_t>(1, atoll(genv)) * mstep : raster_rows(m, n, k, mstep);
      for (int64_t i0 = 0; i0 < m; i0 += group)
        for (int64_t j = 0; j < n; j += tn)
          for (int64_t i = i0; i < std::min(m, i0 + group); i += mstep) push(i, j, false);
    }
    ficco_plan_desc d{};
    d.n_tiles = int32_t(tiles.size());
    d.tiles = tiles.data();
    d.grid = grid;
    d.alpha = 1.0f;
    d.k = k;
    d.tile_n = tn;
    d.cta_group = cta_group;
    ficco_plan* p;
    if ((r = ficco_plan_create(cm, &d, &p))) return r;
    it = cache.emplace(key, std::make_pair(cm, p)).first;
  }
  ficco_plan* p = it->second.second;
  p->desc.a = ficco_operand{FICCO_BUF_A, 0, 0, 0, m, k};
  p->desc.b = ficco_operand{FICCO_BUF_B, 0, 0, 0, n, k};
  p->desc.c = ficco_operand{FICCO_BUF_C, 0, 0, 0, m, n};
  p->desc.k = k;
  p->epi_bufs = epi_bufs_for(k);
  const float prev_alpha = p->desc.alpha;
  const uint32_t prev_hints = p->desc.hints;
  p->desc.alpha = alpha;
  {
    const char* env = getenv("FICCO_A_EVICT_LAST");  // "0" / "1" override the size rule (A/B experiments)
    // column-major rasters (row groups, see raster_rows) keep the group's A slice in L2 and stream B
    const bool grouped = raster_rows(m, n, k, int64_t(ficco::BM) * cta_group) > int64_t(ficco::BM) * cta_group &&
                         epi_bufs_for(k) == 1;
    const bool pin = env && env[0] != 'a' ? env[0] == '1' : (m * k * 2 <= (int64_t(32) << 20) || grouped);
    // W stays evict_last even beyond L2: every column tile is re-read by the group's row blocks, and
    // evict_first lost those hits (2.3-4.6 % slower on C3 G2/G4, C3', EP; r02_experiments/w_policy_ab.json)
    p->desc.hints = pin ? FICCO_HINT_A_EVICT_LAST : 0;
  }
  if (p->desc.alpha != prev_alpha || p->desc.hints != prev_hints)  // the cached kernel params bake both in
    p->pcache[0].valid = p->pcache[1].valid = false;
  return ficco_plan_run_parts(p, a, b, c, stream, 0, 1);  // no flags: direct launch
}

int ficco_gemm_bf16(const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k, float alpha, int grid,
                    void* stream) {
  return ficco_gemm_bf16_cfg(a, b, c, m, n, k, alpha, grid, 0, 0, stream);
}

}  // extern "C"

// ---------------------------------------------------------------- NVLS multicast (comm_agent = nvls)

namespace {
struct McObj {
  CUmemGenericAllocationHandle handle = 0;  // the multicast object
  CUmemGenericAllocationHandle mem = 0;     // this device's backing memory
  size_t bytes = 0, gran = 0;
  CUdeviceptr uc = 0, va = 0;
  bool owner_created = false;
};

int mc_fail(const ficco::McDriver* d, CUresult r, const char* what) {
  const char* s = nullptr;
  if (d->error_string) d->error_string(r, &s);
  return fail(FICCO_ENODEV, std::string(what) + ": " + (s ? s : "CUresult " + std::to_string(int(r))) +
                                " (NVLS multicast unavailable: the comm_agent='nvls' path needs NVSwitch "
                                "multicast access on every rank's GPU)");
}

int mc_prop(const ficco::McDriver* d, size_t bytes, int ndev, CUmulticastObjectProp* prop, size_t* gran) {
  *prop = CUmulticastObjectProp{};
  prop->numDevices = unsigned(ndev);
  prop->handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop->size = 2 << 20;
  CUresult r = d->granularity(gran, prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS || *gran == 0) return mc_fail(d, r, "cuMulticastGetGranularity");
  prop->size = (bytes + *gran - 1) / *gran * *gran;
  return 0;
}
}  // namespace

extern "C" {

int ficco_mc_supported(int device, int* supported) {
  if (!supported) return fail(FICCO_EINVAL, "null argument");
  *supported = 0;
  const ficco::McDriver* d = ficco::mc_driver();
  if (!d->ok) return 0;
  int attr = 0;
  if (d->dev_attr(&attr, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, device) != CUDA_SUCCESS || !attr) return 0;
  // the attribute can be set where the fabric still refuses objects (e.g. a container without the
  // NVSwitch fabric manager): try one
  CUmulticastObjectProp prop;
  size_t gran;
  if (mc_prop(d, 2 << 20, 1, &prop, &gran)) return 0;
  CUmemGenericAllocationHandle h;
  if (d->create(&h, &prop) != CUDA_SUCCESS) return 0;
  d->mem_release(h);
  *supported = 1;
  return 0;
}

int ficco_mc_create(size_t bytes, int n_devices, void** mc, size_t* mapped_bytes) {
  if (!mc || n_devices < 1 || bytes == 0) return fail(FICCO_EINVAL, "bad multicast arguments");
  const ficco::McDriver* d = ficco::mc_driver();
  if (!d->ok) return fail(FICCO_ENODEV, "CUDA driver multicast entry points unavailable");
  CUmulticastObjectProp prop;
  auto* o = new McObj();
  int r = mc_prop(d, bytes, n_devices, &prop, &o->gran);
  if (!r) {
    CUresult cr = d->create(&o->handle, &prop);
    if (cr != CUDA_SUCCESS) r = mc_fail(d, cr, "cuMulticastCreate");
  }
  if (r) {
    delete o;
    return r;
  }
  o->bytes = prop.size;
  o->owner_created = true;
  if (mapped_bytes) *mapped_bytes = o->bytes;
  *mc = o;
  return 0;
}

int ficco_mc_export(void* mc, int* fd) {
  auto* o = static_cast<McObj*>(mc);
  if (!o || !fd) return fail(FICCO_EINVAL, "null argument");
  const ficco::McDriver* d = ficco::mc_driver();
  CUresult r = d->export_handle(fd, o->handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  return r == CUDA_SUCCESS ? 0 : mc_fail(d, r, "cuMemExportToShareableHandle");
}

int ficco_mc_import(int fd, size_t mapped_bytes, void** mc) {
  if (!mc || fd < 0 || mapped_bytes == 0) return fail(FICCO_EINVAL, "bad multicast import arguments");
  const ficco::McDriver* d = ficco::mc_driver();
  if (!d->ok) return fail(FICCO_ENODEV, "CUDA driver multicast entry points unavailable");
  auto* o = new McObj();
  CUresult r = d->import_handle(&o->handle, reinterpret_cast<void*>(uintptr_t(fd)),
                                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    delete o;
    return mc_fail(d, r, "cuMemImportFromShareableHandle");
  }
  o->bytes = mapped_bytes;
  *mc = o;
  return 0;
}

int ficco_mc_add_device(void* mc) {
  auto* o = static_cast<McObj*>(mc);
  if (!o) return fail(FICCO_EINVAL, "null multicast object");
  const ficco::McDriver* d = ficco::mc_driver();
  CUdevice dev;
  CUresult r = d->ctx_get_device(&dev);
  if (r == CUDA_SUCCESS) r = d->add_device(o->handle, dev);
  return r == CUDA_SUCCESS ? 0 : mc_fail(d, r, "cuMulticastAddDevice");
}

int ficco_mc_bind(void* mc, void** uc_va, void** mc_va) {
  auto* o = static_cast<McObj*>(mc);
  if (!o || !uc_va || !mc_va) return fail(FICCO_EINVAL, "null argument");
  const ficco::McDriver* d = ficco::mc_driver();
  CUdevice dev;
  CUresult r = d->ctx_get_device(&dev);
  if (r != CUDA_SUCCESS) return mc_fail(d, r, "cuCtxGetDevice");
  if (!o->gran) {
    CUmulticastObjectProp prop;
    if (int e = mc_prop(d, o->bytes, 1, &prop, &o->gran)) return e;
  }
  CUmemAllocationProp mp{};
  mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  mp.location.id = dev;
  mp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if ((r = d->mem_create(&o->mem, o->bytes, &mp, 0)) != CUDA_SUCCESS) return mc_fail(d, r, "cuMemCreate");
  if ((r = d->bind_mem(o->handle, 0, o->mem, 0, o->bytes, 0)) != CUDA_SUCCESS)
    return mc_fail(d, r, "cuMulticastBindMem");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((r = d->reserve(&o->uc, o->bytes, o->gran, 0, 0)) != CUDA_SUCCESS ||
      (r = d->map(o->uc, o->bytes, 0, o->mem, 0)) != CUDA_SUCCESS ||
      (r = d->set_access(o->uc, o->bytes, &acc, 1)) != CUDA_SUCCESS ||
      (r = d->reserve(&o->va, o->bytes, o->gran, 0, 0)) != CUDA_SUCCESS ||
      (r = d->map(o->va, o->bytes, 0, o->handle, 0)) != CUDA_SUCCESS ||
      (r = d->set_access(o->va, o->bytes, &acc, 1)) != CUDA_SUCCESS)
    return mc_fail(d, r, "mapping the multicast workspace");
  *uc_va = reinterpret_cast<void*>(o->uc);
  *mc_va = reinterpret_cast<void*>(o->va);
  return 0;
}

int ficco_mc_release(void* mc) {
  auto* o = static_cast<McObj*>(mc);
  if (!o) return 0;
  const ficco::McDriver* d = ficco::mc_driver();
  if (o->va) {
    d->unmap(o->va, o->bytes);
    d->addr_free(o->va, o->bytes);
  }
  if (o->uc) {
    d->unmap(o->uc, o->bytes);
    d->addr_free(o->uc, o->bytes);
  }
  if (o->mem) d->mem_release(o->mem);
  if (o->handle) d->mem_release(o->handle);
  delete o;
  return 0;
}

int ficco_comm_set_multicast(ficco_comm_t* c, void* uc_va, void* mc_va, size_t bytes) {
  if (!c) return fail(FICCO_EINVAL, "null comm");
  c->mc_uc = static_cast<uint8_t*>(uc_va);
  c->mc_va = static_cast<uint8_t*>(mc_va);
  c->mc_bytes = uc_va && mc_va ? bytes : 0;
  return 0;
}

int ficco_mc_reduce_bf16(const void* mc_src, void* dst, int64_t rows, int64_t cols, int64_t ld_src, int64_t ld_dst,
                         void* stream) {
  if (!mc_src || !dst || rows <= 0 || cols <= 0 || cols % 8 || ld_src % 8 || ld_dst % 8)
    return fail(FICCO_EINVAL, "mc_reduce: 16-byte rows (cols, ld multiples of 8) required");
  int dev, sms;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t vecs = rows * (cols / 8);
  const int grid = int(std::min<int64_t>(std::max<int64_t>(1, (vecs + 255) / 256), 4 * sms));
  ficco::mc_reduce_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(mc_src), static_cast<uint8_t*>(dst), rows, cols * 2, ld_src * 2, ld_dst * 2);
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"

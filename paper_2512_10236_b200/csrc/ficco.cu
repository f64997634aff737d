// libficco_b200: C-ABI executor for lowered FiCCO plans on B200 (sm_100a).
//
// Host side of the executor declared in include/ficco.h. Responsibilities:
//   * symmetric workspace + CUDA IPC plumbing (ranks exchange handles in Python),
//   * the copy program: copy-engine copies batched per round with
//     cudaMemcpyBatchAsync (1D) / cudaMemcpy2DAsync (2D slabs) on a dedicated
//     copy stream, stream memory operations (cuStreamWriteValue32 /
//     cuStreamWaitValue32) for readiness flags — no SMs, no host round trips,
//   * the tile program: TMA descriptors + one persistent tcgen05 kernel launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ficco.h"
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

struct Driver {
  PFN_encodeTiled encode = nullptr;
  PFN_writeValue32 write32 = nullptr;
  PFN_waitValue32 wait32 = nullptr;
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
              get("cuStreamWaitValue32", reinterpret_cast<void**>(&d.wait32));
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

int g_kernel_configured = -1;  // device id the kernel attributes were set for

int configure_kernel(int dev) {
  if (g_kernel_configured == dev) return 0;
  CK(cudaFuncSetAttribute(ficco::tile_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          ficco::SMEM_BYTES));
  g_kernel_configured = dev;
  return 0;
}

}  // namespace

struct ficco_comm {
  int rank = 0, world = 1, device = 0, sms = 0;
  bool virt = false;
  size_t ws_bytes = 0;
  std::vector<uint8_t*> ws;  // per rank, mapped into this process
  std::vector<void*> owned;  // virtual-mode peer workspaces we allocated
  uint32_t epoch = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_counters = nullptr;
  Driver* drv = nullptr;
  uint32_t* flags(int r) { return reinterpret_cast<uint32_t*>(ws[r]); }
};

struct ficco_plan {
  ficco_comm* comm = nullptr;
  std::vector<ficco_copy_op> ops;
  ficco_tile* d_tiles = nullptr;
  int n_tiles = 0;
  ficco_plan_desc desc{};
};

namespace {

int resolve(ficco_comm* c, int buf, int peer, int64_t off, int64_t par, const void* a, const void* b, void* cc,
            uint8_t** out) {
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
    default: return fail(FICCO_EINVAL, "bad buffer id " + std::to_string(buf));
  }
  if (!base) return fail(FICCO_EINVAL, "null buffer for id " + std::to_string(buf));
  *out = base + off + ((c->epoch & 1u) ? par : 0);
  return 0;
}

struct Batch {
  std::vector<void*> dst;
  std::vector<void*> src;
  std::vector<size_t> size;
};

int flush(Batch& b, cudaStream_t s) {
  if (b.dst.empty()) return 0;
  cudaMemcpyAttributes attr{};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
  size_t idx = 0, fail_idx = 0;
  cudaError_t e = cudaMemcpyBatchAsync(b.dst.data(), b.src.data(), b.size.data(), b.dst.size(), &attr, &idx, 1,
                                       &fail_idx, s);
  if (e != cudaSuccess) {
    // Older drivers: fall back to one cudaMemcpyAsync per copy (still copy engines).
    cudaGetLastError();
    for (size_t i = 0; i < b.dst.size(); ++i)
      CK(cudaMemcpyAsync(b.dst[i], b.src[i], b.size[i], cudaMemcpyDefault, s));
  }
  b.dst.clear();
  b.src.clear();
  b.size.clear();
  return 0;
}

int run_copy_program(ficco_plan* p, const void* a, const void* b, void* c) {
  ficco_comm* cm = p->comm;
  Batch batch;
  const uint32_t epoch = cm->epoch;
  for (const ficco_copy_op& op : p->ops) {
    switch (op.op) {
      case FICCO_OP_COPY: {
        uint8_t *src, *dst;
        int r = resolve(cm, op.src_buf, op.peer, op.src_off, op.src_par, a, b, c, &src);
        if (r) return r;
        r = resolve(cm, op.dst_buf, op.dst_peer, op.dst_off, op.dst_par, a, b, c, &dst);
        if (r) return r;
        if (op.height <= 1) {
          batch.dst.push_back(dst);
          batch.src.push_back(src);
          batch.size.push_back(size_t(op.width));
        } else {
          if ((r = flush(batch, cm->copy))) return r;
          CK(cudaMemcpy2DAsync(dst, size_t(op.dst_pitch), src, size_t(op.src_pitch), size_t(op.width),
                               size_t(op.height), cudaMemcpyDefault, cm->copy));
        }
        break;
      }
      case FICCO_OP_SIGNAL: {
        int r = flush(batch, cm->copy);
        if (r) return r;
        CKD(cm->drv->write32(cm->copy, CUdeviceptr(cm->flags(cm->rank) + op.flag), epoch, 0));
        break;
      }
      case FICCO_OP_NOTIFY: {
        int r = flush(batch, cm->copy);
        if (r) return r;
        if (op.peer < 0 || op.peer >= cm->world) return fail(FICCO_EINVAL, "notify peer out of range");
        if (!cm->virt) CKD(cm->drv->write32(cm->copy, CUdeviceptr(cm->flags(op.peer) + op.flag), epoch, 0));
        break;
      }
      case FICCO_OP_WAIT: {
        int r = flush(batch, cm->copy);
        if (r) return r;
        // wait until flag >= epoch - value (value = epoch lag, e.g. 1 for "peer finished the previous run")
        if (!cm->virt)
          CKD(cm->drv->wait32(cm->copy, CUdeviceptr(cm->flags(cm->rank) + op.flag), epoch - op.value,
                              CU_STREAM_WAIT_VALUE_GEQ));
        break;
      }
      case FICCO_OP_WAIT_COUNTER: {
        int r = flush(batch, cm->copy);
        if (r) return r;
        CKD(cm->drv->wait32(cm->copy, CUdeviceptr(cm->flags(cm->rank) + FICCO_FLAG_COUNTERS + op.flag), op.value,
                            CU_STREAM_WAIT_VALUE_GEQ));
        break;
      }
      default: return fail(FICCO_EINVAL, "bad copy opcode " + std::to_string(op.op));
    }
  }
  return flush(batch, cm->copy);
}

int launch_tiles(ficco_plan* p, const void* a, const void* b, void* c, cudaStream_t s) {
  ficco_comm* cm = p->comm;
  const ficco_plan_desc& d = p->desc;
  if (p->n_tiles == 0) return 0;
  int r = configure_kernel(cm->device);
  if (r) return r;
  ficco::TileParams prm;
  memset(&prm, 0, sizeof(prm));
  uint8_t* pa;
  uint8_t* pb;
  if ((r = resolve(cm, d.a.buf, -1, d.a.off, d.a.par, a, b, c, &pa))) return r;
  if ((r = resolve(cm, d.b.buf, -1, d.b.off, d.b.par, a, b, c, &pb))) return r;
  if ((r = encode_bf16_2d(cm->drv, &prm.tmap_a, pa, d.a.rows, d.k, d.a.ld, ficco::BM))) return r;
  if ((r = encode_bf16_2d(cm->drv, &prm.tmap_b, pb, d.b.rows, d.k, d.b.ld, ficco::BN))) return r;
  uint8_t* po = nullptr;
  if (d.c.buf != FICCO_BUF_NONE && (r = resolve(cm, d.c.buf, -1, d.c.off, d.c.par, a, b, c, &po))) return r;
  uint8_t* pp = nullptr;
  if (d.part.buf != FICCO_BUF_NONE && (r = resolve(cm, d.part.buf, -1, d.part.off, d.part.par, a, b, c, &pp)))
    return r;
  prm.tiles = p->d_tiles;
  prm.num_tiles = p->n_tiles;
  prm.num_kb = int((d.k + ficco::BK - 1) / ficco::BK);
  prm.out = reinterpret_cast<__nv_bfloat16*>(po);
  prm.part = reinterpret_cast<__nv_bfloat16*>(pp);
  prm.ld_out = d.c.ld;
  prm.ld_part = d.part.ld;
  prm.n_recv = d.n_recv;
  for (int j = 0; j < d.n_recv; ++j) {
    uint8_t* pr;
    if ((r = resolve(cm, d.recv.buf, -1, d.recv.off + j * d.recv_slot, d.recv.par, a, b, c, &pr))) return r;
    prm.recv[j] = reinterpret_cast<const __nv_bfloat16*>(pr);
  }
  prm.ld_recv = d.recv.ld;
  prm.rs_flag0 = d.rs_flag0;
  prm.flags = cm->flags(cm->rank);
  prm.counters = prm.flags + FICCO_FLAG_COUNTERS;
  prm.abort_word = prm.flags + FICCO_FLAG_ABORT;
  prm.epoch = cm->epoch;
  prm.alpha = d.alpha;
  int grid = d.grid > 0 ? d.grid : cm->sms;
  if (grid > p->n_tiles) grid = p->n_tiles;
  ficco::tile_gemm_kernel<<<grid, ficco::NUM_THREADS, ficco::SMEM_BYTES, s>>>(prm);
  CK(cudaGetLastError());
  return 0;
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
  cudaError_t e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_counters, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete c;
    return fail(FICCO_ECUDA, std::string("comm stream/event creation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return 0;
}

int ficco_comm_destroy(ficco_comm_t* c) {
  if (!c) return 0;
  cudaStreamSynchronize(c->copy);
  cudaStreamDestroy(c->copy);
  cudaEventDestroy(c->ev_fork);
  cudaEventDestroy(c->ev_join);
  cudaEventDestroy(c->ev_counters);
  delete c;
  return 0;
}

int ficco_comm_epoch(ficco_comm_t* c, uint32_t* epoch) {
  if (!c || !epoch) return fail(FICCO_EINVAL, "null argument");
  *epoch = c->epoch;
  return 0;
}

int ficco_comm_check(ficco_comm_t* c, void* stream) {
  if (!c) return fail(FICCO_EINVAL, "null comm");
  CK(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
  CK(cudaStreamSynchronize(c->copy));
  uint32_t abort_word = 0;
  CK(cudaMemcpy(&abort_word, c->flags(c->rank) + FICCO_FLAG_ABORT, 4, cudaMemcpyDeviceToHost));
  if (abort_word) return fail(FICCO_ETIMEOUT, "tile kernel timed out waiting for a readiness flag");
  return 0;
}

int ficco_comm_set_flags(ficco_comm_t* c, int first, int count, uint32_t value, void* stream) {
  if (!c || first < 0 || count < 0 || first + count > FICCO_WS_FLAG_WORDS) return fail(FICCO_EINVAL, "bad flag range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < count; ++i)
    CKD(c->drv->write32(s, CUdeviceptr(c->flags(c->rank) + first + i), value, 0));
  return 0;
}

int ficco_plan_create(ficco_comm_t* c, const ficco_plan_desc* d, ficco_plan_t** out) {
  if (!c || !d || !out) return fail(FICCO_EINVAL, "null argument");
  if (d->n_tiles < 0 || d->n_ops < 0) return fail(FICCO_EINVAL, "negative program length");
  if (d->n_tiles > 0 && (d->k <= 0 || d->k % 8 != 0)) return fail(FICCO_EINVAL, "K must be a positive multiple of 8");
  if (d->n_recv < 0 || d->n_recv > ficco::MAX_RECV) return fail(FICCO_EINVAL, "too many receive slots");
  if (d->n_counters < 0 || FICCO_FLAG_COUNTERS + d->n_counters >= FICCO_FLAG_ABORT)
    return fail(FICCO_EINVAL, "too many counters");
  for (int i = 0; i < d->n_tiles; ++i) {
    const ficco_tile& t = d->tiles[i];
    if (t.rows < 1 || t.rows > ficco::BM || t.cols < 32 || t.cols > ficco::BN || t.cols % 32)
      return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": rows/cols out of range");
    if (t.mode < FICCO_EPI_STORE || t.mode > FICCO_EPI_REDUCE)
      return fail(FICCO_EINVAL, "tile " + std::to_string(i) + ": bad epilogue mode");
    if (t.flag >= FICCO_FLAG_COUNTERS) return fail(FICCO_EINVAL, "tile flag index out of range");
  }
  auto* p = new ficco_plan();
  p->comm = c;
  p->desc = *d;
  p->ops.assign(d->ops, d->ops + d->n_ops);
  p->desc.ops = nullptr;
  p->desc.tiles = nullptr;
  p->n_tiles = d->n_tiles;
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
  if (p->d_tiles) cudaFree(p->d_tiles);
  delete p;
  return 0;
}

int ficco_plan_run_parts(ficco_plan_t* p, const void* a, const void* b, void* c, void* stream, int run_copies,
                         int run_tiles) {
  if (!p) return fail(FICCO_EINVAL, "null plan");
  ficco_comm* cm = p->comm;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cm->epoch += 1;
  int r;
  // counters are per-run: reset them on the compute stream before anything waits on them
  if (p->desc.n_counters > 0) {
    CK(cudaMemsetAsync(cm->flags(cm->rank) + FICCO_FLAG_COUNTERS, 0, 4 * size_t(p->desc.n_counters), s));
  }
  const bool copies = run_copies && !p->ops.empty();
  if (copies) {
    CK(cudaEventRecord(cm->ev_fork, s));
    CK(cudaStreamWaitEvent(cm->copy, cm->ev_fork, 0));
  }
  if (run_tiles && (r = launch_tiles(p, a, b, c, s))) return r;
  if (copies) {
    if ((r = run_copy_program(p, a, b, c))) return r;
    CK(cudaEventRecord(cm->ev_join, cm->copy));
    CK(cudaStreamWaitEvent(s, cm->ev_join, 0));
  }
  return 0;
}

int ficco_plan_run(ficco_plan_t* p, const void* a, const void* b, void* c, void* stream) {
  return ficco_plan_run_parts(p, a, b, c, stream, 1, 1);
}

int ficco_copy_batch(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t count, void* stream) {
  Batch b;
  for (size_t i = 0; i < count; ++i) {
    b.dst.push_back(dsts[i]);
    b.src.push_back(const_cast<void*>(srcs[i]));
    b.size.push_back(sizes[i]);
  }
  return flush(b, reinterpret_cast<cudaStream_t>(stream));
}

int ficco_gemm_bf16(const void* a, const void* b, void* c, int64_t m, int64_t n, int64_t k, float alpha, int grid,
                    void* stream) {
  // Plain C = alpha * A @ B^T through the same tile kernel (no flags), cached per shape.
  if (m <= 0 || n <= 0 || k <= 0 || n % 32 || k % 8) return fail(FICCO_EINVAL, "gemm: need N%32==0, K%8==0");
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int, int>, std::pair<ficco_comm*, ficco_plan*>> cache;
  std::lock_guard<std::mutex> lock(mu);
  int dev;
  CK(cudaGetDevice(&dev));
  auto key = std::make_tuple(m, n, grid, dev);
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
    std::vector<ficco_tile> tiles;
    for (int64_t i = 0; i < m; i += ficco::BM)
      for (int64_t j = 0; j < n; j += ficco::BN) {
        ficco_tile t{};
        t.a_row = int32_t(i);
        t.b_row = int32_t(j);
        t.c_row = int32_t(i);
        t.c_col = int32_t(j);
        t.rows = int16_t(m - i < ficco::BM ? m - i : ficco::BM);
        t.cols = int16_t(n - j < ficco::BN ? n - j : ficco::BN);
        t.flag = -1;
        t.mode = FICCO_EPI_STORE;
        tiles.push_back(t);
      }
    ficco_plan_desc d{};
    d.n_tiles = int32_t(tiles.size());
    d.tiles = tiles.data();
    d.grid = grid;
    d.alpha = 1.0f;
    d.k = k;
    ficco_plan* p;
    if ((r = ficco_plan_create(cm, &d, &p))) return r;
    it = cache.emplace(key, std::make_pair(cm, p)).first;
  }
  ficco_plan* p = it->second.second;
  p->desc.a = ficco_operand{FICCO_BUF_A, 0, 0, 0, m, k};
  p->desc.b = ficco_operand{FICCO_BUF_B, 0, 0, 0, n, k};
  p->desc.c = ficco_operand{FICCO_BUF_C, 0, 0, 0, m, n};
  p->desc.k = k;
  p->desc.alpha = alpha;
  return ficco_plan_run_parts(p, a, b, c, stream, 0, 1);
}

}  // extern "C"

// Write-only HBM bandwidth ceiling on this B200 (the C4 score write's roofline denominator).
//
// torch fill_/zero_ reach only ~3.9 TB/s, below what the tile kernel's TMA-store epilogue
// already sustains, so they are not the ceiling. This probe streams 4 GiB of writes with
// the store flavours an epilogue can use and reports the best:
//   v4      st.global.v4.b32            (16 B per thread, plain)
//   v4cs    st.global.cs.v4.b32         (streaming / evict-first)
//   v8      st.global.v8.b32            (32 B per thread, sm_100 256-bit stores)
//   bulk    cp.async.bulk.global.shared::cta (TMA bulk store of a 4 KiB smem buffer per warp)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_write_probe tools/hbm_write_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void w_v4(uint4* p, int64_t n16) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void w_v4cs(uint4* p, int64_t n16) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(p + i), "r"(int(threadIdx.x)) : "memory");
}

__global__ void w_v8(uint4* p, int64_t n16) {
  const int64_t n32 = n16 / 2;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n32; i += int64_t(gridDim.x) * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(p + 2 * i), "r"(int(threadIdx.x))
                 : "memory");
}

// each warp owns a 4 KiB smem buffer and issues one bulk store per 4 KiB chunk, keeping
// up to DEPTH bulk groups in flight (the tile kernel's epilogue pattern without the math)
template <int DEPTH>
__global__ void w_bulk(uint8_t* p, int64_t nbytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* buf = sm + warp * 4096;
  for (int i = lane; i < 4096 / 16; i += 32) reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, warp, 1, 2);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t chunks = nbytes / 4096;
  const int64_t wid = blockIdx.x * int64_t(blockDim.x / 32) + warp;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x / 32);
  if (lane == 0) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    for (int64_t c = wid; c < chunks; c += nw) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(p + c * 4096), "r"(s)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

template <class F>
static double best_gbps(F launch, int64_t bytes, float* med) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  std::vector<float> ms;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  *med = float(bytes / (ms[ms.size() / 2] * 1e-3) / 1e9);
  return bytes / (ms[0] * 1e-3) / 1e9;
}

int main() {
  const int64_t bytes = int64_t(4) << 30;
  uint8_t* p;
  CK(cudaMalloc(&p, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n16 = bytes / 16;
  std::printf("{");
  const char* sep = "";
  auto report = [&](const char* name, double best, float med) {
    std::printf("%s\"%s\": {\"best_GBps\": %.1f, \"median_GBps\": %.1f}", sep, name, best, med);
    sep = ", ";
  };
  for (int per_sm : {4, 8, 16}) {
    float med;
    char name[32];
    double b = best_gbps([&] { w_v4<<<sms * per_sm, 256>>>(reinterpret_cast<uint4*>(p), n16); }, bytes, &med);
    std::snprintf(name, sizeof name, "v4_x%d", per_sm);
    report(name, b, med);
    b = best_gbps([&] { w_v4cs<<<sms * per_sm, 256>>>(reinterpret_cast<uint4*>(p), n16); }, bytes, &med);
    std::snprintf(name, sizeof name, "v4cs_x%d", per_sm);
    report(name, b, med);
    b = best_gbps([&] { w_v8<<<sms * per_sm, 256>>>(reinterpret_cast<uint4*>(p), n16); }, bytes, &med);
    std::snprintf(name, sizeof name, "v8_x%d", per_sm);
    report(name, b, med);
  }
  CK(cudaFuncSetAttribute(w_bulk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
  CK(cudaFuncSetAttribute(w_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
  CK(cudaFuncSetAttribute(w_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
  for (int per_sm : {1, 2, 4}) {
    float med;
    char name[32];
    double b = best_gbps([&] { w_bulk<1><<<sms * per_sm, 256, 8 * 4096>>>(p, bytes); }, bytes, &med);
    std::snprintf(name, sizeof name, "bulk_d1_x%d", per_sm);
    report(name, b, med);
    b = best_gbps([&] { w_bulk<2><<<sms * per_sm, 256, 8 * 4096>>>(p, bytes); }, bytes, &med);
    std::snprintf(name, sizeof name, "bulk_d2_x%d", per_sm);
    report(name, b, med);
    b = best_gbps([&] { w_bulk<4><<<sms * per_sm, 256, 8 * 4096>>>(p, bytes); }, bytes, &med);
    std::snprintf(name, sizeof name, "bulk_d4_x%d", per_sm);
    report(name, b, med);
  }
  std::printf("}\n");
  CK(cudaGetLastError());
  return 0;
}

// Does this box expose NVLS multicast to a one-GPU process? Creates a multicast object with one device,
// binds device memory to it, maps the multicast VA, and checks multimem.ld_reduce (bf16x2, f32 accumulate)
// and multimem.st against plain loads of the backing memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CKD(x)                                                                         \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s = nullptr;                                                         \
      cuGetErrorString(r_, &s);                                                        \
      std::printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s ? s : "?");      \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void reduce_kernel(const __nv_bfloat16* mc, __nv_bfloat16* out, int n2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  uint32_t v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.bf16x2 %0, [%1];"
               : "=r"(v)
               : "l"(reinterpret_cast<const uint32_t*>(mc) + i)
               : "memory");
  reinterpret_cast<uint32_t*>(out)[i] = v;
}

__global__ void store_kernel(__nv_bfloat16* mc, int n2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  __nv_bfloat162 h = __floats2bfloat162_rn(float(i % 97), 0.5f);
  asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(reinterpret_cast<uint32_t*>(mc) + i),
               "r"(*reinterpret_cast<uint32_t*>(&h))
               : "memory");
}

int main() {
  CKD(cuInit(0));
  CUdevice dev;
  CKD(cuDeviceGet(&dev, 0));
  int mc_ok = 0;
  CKD(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  std::printf("{\"multicast_supported\": %d}\n", mc_ok);
  if (!mc_ok) return 0;
  CUcontext ctx;
  CKD(cuDevicePrimaryCtxRetain(&ctx, dev));
  CKD(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp prop{};
  size_t gran = 0;
  size_t bytes = 0;
  CUmemGenericAllocationHandle mc;
  {  // which (handle type, device count) combinations does the driver accept here?
    const CUmemAllocationHandleType types[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                               CU_MEM_HANDLE_TYPE_FABRIC};
    const char* tn[] = {"posix_fd", "none", "fabric"};
    bool made = false;
    for (int ti = 0; ti < 3 && !made; ++ti)
      for (int nd : {1, 2}) {
        CUmulticastObjectProp pr{};
        pr.numDevices = nd;
        pr.handleTypes = types[ti];
        pr.size = 2 << 20;
        size_t g = 0;
        CUresult rg = cuMulticastGetGranularity(&g, &pr, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        if (rg != CUDA_SUCCESS || g == 0) {
          std::printf("{\"handle\": \"%s\", \"devices\": %d, \"granularity_error\": %d}\n", tn[ti], nd, int(rg));
          continue;
        }
        pr.size = ((size_t(64) << 20) + g - 1) / g * g;
        CUresult rc = cuMulticastCreate(&mc, &pr);
        std::printf("{\"handle\": \"%s\", \"devices\": %d, \"granularity\": %zu, \"create\": %d}\n", tn[ti], nd, g,
                    int(rc));
        if (rc == CUDA_SUCCESS) {
          if (nd == 1) {
            prop = pr, gran = g, bytes = pr.size, made = true;
            break;
          }
          cuMemRelease(mc);
        }
      }
    if (!made) return 0;
  }
  CKD(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp mp{};
  mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  mp.location.id = 0;
  mp.requestedHandleTypes = CUmemAllocationHandleType(prop.handleTypes);
  CUmemGenericAllocationHandle mem;
  CKD(cuMemCreate(&mem, bytes, &mp, 0));
  CKD(cuMulticastBindMem(mc, 0, mem, 0, bytes, 0));
  CUdeviceptr uc = 0, mcva = 0;
  CKD(cuMemAddressReserve(&uc, bytes, gran, 0, 0));
  CKD(cuMemMap(uc, bytes, 0, mem, 0));
  CKD(cuMemAddressReserve(&mcva, bytes, gran, 0, 0));
  CKD(cuMemMap(mcva, bytes, 0, mc, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CKD(cuMemSetAccess(uc, bytes, &acc, 1));
  CKD(cuMemSetAccess(mcva, bytes, &acc, 1));
  const int n2 = int(bytes / 4);
  store_kernel<<<(n2 + 255) / 256, 256>>>(reinterpret_cast<__nv_bfloat16*>(mcva), n2);
  __nv_bfloat16* out;
  cudaMalloc(&out, bytes);
  reduce_kernel<<<(n2 + 255) / 256, 256>>>(reinterpret_cast<const __nv_bfloat16*>(mcva), out, n2);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    std::printf("{\"kernel_error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  std::vector<uint32_t> a(n2), b(n2);
  cudaMemcpy(a.data(), reinterpret_cast<void*>(uc), bytes, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), out, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n2; ++i) bad += a[i] != b[i];
  // time the multicast ld_reduce read of 64 MiB (one device: a plain read through the switch path)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r)
    reduce_kernel<<<(n2 + 255) / 256, 256>>>(reinterpret_cast<const __nv_bfloat16*>(mcva), out, n2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("{\"multicast_ok\": %d, \"mismatches\": %d, \"words\": %d, \"granularity\": %zu, "
              "\"ld_reduce_GBps\": %.1f}\n",
              bad == 0, bad, n2, gran, 10.0 * bytes / (ms * 1e-3) / 1e9);
  return 0;
}

// NVLS (NVLink SHARP) multicast plumbing and the in-switch reduction kernel (comm_agent = nvls GEMM -> RS).
//
// Every rank binds MC_BYTES of its own HBM to one multicast object; the copy program's REDUCE_MC op then
// reads the owner's rows through the multicast VA with multimem.ld_reduce, so the NVSwitch returns the
// sum over every rank's copy (fp32 accumulation of the bf16 partials, one bf16 rounding). Driver symbols
// are resolved at first use through cudaGetDriverEntryPoint, like the rest of the library, so the .so
// still loads where there is no driver.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace ficco {

// dst rows := sum over the multicast object's devices of the src rows (src is a multicast VA). Each thread
// moves 16 bytes (8 bf16) per step: multimem.ld_reduce ... .v4.bf16x2 with fp32 accumulation in the switch.
__global__ void __launch_bounds__(256) mc_reduce_kernel(const uint8_t* src, uint8_t* dst, int64_t rows,
                                                        int64_t width, int64_t src_pitch, int64_t dst_pitch) {
  const int64_t vec_per_row = width / 16;
  const int64_t total = rows * vec_per_row;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec_per_row, v = i % vec_per_row;
    const uint8_t* s = src + r * src_pitch + v * 16;
    uint32_t x0, x1, x2, x3;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                 : "l"(s)
                 : "memory");
    *reinterpret_cast<uint4*>(dst + r * dst_pitch + v * 16) = make_uint4(x0, x1, x2, x3);
  }
}

struct McDriver {
  CUresult (*create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*add_device)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                       unsigned long long) = nullptr;
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                         unsigned long long) = nullptr;
  CUresult (*mem_release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*export_handle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                            unsigned long long) = nullptr;
  CUresult (*import_handle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*ctx_get_device)(CUdevice*) = nullptr;
  CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*error_string)(CUresult, const char**) = nullptr;
  bool ok = false;
};

inline const McDriver* mc_driver() {
  static McDriver d;
  static bool once = [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
#define FICCO_MC_SYM(field, name) get(name, reinterpret_cast<void**>(&d.field))
    d.ok = FICCO_MC_SYM(create, "cuMulticastCreate") && FICCO_MC_SYM(granularity, "cuMulticastGetGranularity") &&
           FICCO_MC_SYM(add_device, "cuMulticastAddDevice") && FICCO_MC_SYM(bind_mem, "cuMulticastBindMem") &&
           FICCO_MC_SYM(mem_create, "cuMemCreate") && FICCO_MC_SYM(mem_release, "cuMemRelease") &&
           FICCO_MC_SYM(reserve, "cuMemAddressReserve") && FICCO_MC_SYM(addr_free, "cuMemAddressFree") &&
           FICCO_MC_SYM(map, "cuMemMap") && FICCO_MC_SYM(unmap, "cuMemUnmap") &&
           FICCO_MC_SYM(set_access, "cuMemSetAccess") &&
           FICCO_MC_SYM(export_handle, "cuMemExportToShareableHandle") &&
           FICCO_MC_SYM(import_handle, "cuMemImportFromShareableHandle") &&
           FICCO_MC_SYM(ctx_get_device, "cuCtxGetDevice") && FICCO_MC_SYM(dev_attr, "cuDeviceGetAttribute") &&
           FICCO_MC_SYM(error_string, "cuGetErrorString");
#undef FICCO_MC_SYM
    return true;
  }();
  (void)once;
  return &d;
}

}  // namespace ficco

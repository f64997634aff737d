// comm_agent = core: a transfer executed by SMs (P2P loads / stores over NVLink, or local
// HBM for virtual peers) instead of a copy engine — the paper's "core-driven" communication
// (reference machines.py:48 comm_agent 'core', engine.py:128 CIL multipliers for it), kept as
// the contention comparison point for the copy-engine path.
//
// Small (256 threads, <= 64 registers, no shared memory) so it co-resides with the persistent
// tile kernel, whose register cap leaves exactly this room (tile_kernel.cuh MAX_REGS): the
// copy then competes with the GEMM for issue slots, L2 and HBM, which is what the variant
// measures. 16-byte vectors, 4 in flight per thread.
#pragma once

#include <cstdint>

namespace ficco {

constexpr int COPY_THREADS = 256;
constexpr int COPY_UNROLL = 4;

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// rows x width bytes, row pitches in bytes; 16-byte aligned addresses, widths and pitches.
__global__ void __launch_bounds__(COPY_THREADS, 4)
    sm_copy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t width, int64_t height,
                   int64_t src_pitch, int64_t dst_pitch) {
  const int64_t per_row = width >> 4;
  const int64_t total = per_row * height;
  const int64_t stride = int64_t(gridDim.x) * COPY_THREADS;
  int64_t i = int64_t(blockIdx.x) * COPY_THREADS + threadIdx.x;
  for (; i + (COPY_UNROLL - 1) * stride < total; i += COPY_UNROLL * stride) {
    uint4 v[COPY_UNROLL];
#pragma unroll
    for (int u = 0; u < COPY_UNROLL; ++u) {
      const int64_t e = i + u * stride, r = e / per_row, c = e - r * per_row;
      v[u] = ld_nc_v4(reinterpret_cast<const uint4*>(src + r * src_pitch) + c);
    }
#pragma unroll
    for (int u = 0; u < COPY_UNROLL; ++u) {
      const int64_t e = i + u * stride, r = e / per_row, c = e - r * per_row;
      reinterpret_cast<uint4*>(dst + r * dst_pitch)[c] = v[u];
    }
  }
  for (; i < total; i += stride) {
    const int64_t r = i / per_row, c = i - r * per_row;
    reinterpret_cast<uint4*>(dst + r * dst_pitch)[c] = ld_nc_v4(reinterpret_cast<const uint4*>(src + r * src_pitch) + c);
  }
}

}  // namespace ficco

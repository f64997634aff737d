// Epilogue data-path probe: what bounds the C4 score-write kernel (TMEM -> regs -> smem -> TMA store)?
//
// 148 persistent CTAs x 320 threads (the tile kernel's shape), 512 TMEM columns, 8 epilogue warps with
// EB = 3 staging buffers each, output [16384, 131072] bf16 (C4's 4 GiB score matrix), 128 x 256 tiles per
// CTA in row-major tile order. No MMA: TMEM holds whatever it holds. Modes:
//   ldtm    tcgen05.ld 32x32b.x32 + wait only (the TMEM read stream)
//   sts     pack + st.shared (swizzled) only
//   tma     st.shared + TMA tensor stores (no TMEM reads)
//   ldsts   LDTM + st.shared (no stores to global)
//   full    LDTM + st.shared + TMA stores: the epilogue without the MMA
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/epi_probe tools/epi_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_2512_10236_b200/csrc/sm100_primitives.cuh"

using namespace ficco;

constexpr int TQ = 16384, TKV = 131072, TMR = 128, TNC = 256, EB = 3;
constexpr int NT = 320;

enum { M_LDTM = 0, M_STS = 1, M_TMA = 2, M_LDSTS = 3, M_FULL = 4 };
// loads: 0 none; 1 A and B boxes per tile (the tile kernel's operand traffic: 2 k-blocks of a 128-row
// A box and a 128-row B box, 64 KB per tile per CTA); 2 B only (A stationary: 32 KB per tile)
constexpr int LSTAGES = 3, LSTAGE_BYTES = 2 * 128 * 64 * 2;

__device__ __forceinline__ uint32_t swz128(uint32_t t, uint32_t j) { return t * 128u + ((j ^ (t & 7u)) << 4); }

__global__ void __launch_bounds__(NT, 1) probe(const __grid_constant__ CUtensorMap out_map,
                                                const __grid_constant__ CUtensorMap a_map,
                                                const __grid_constant__ CUtensorMap b_map, int mode, int tiles,
                                                uint32_t* sink, int hint_kind, int order, int loads,
                                                const __grid_constant__ CUtensorMap out3_map, int wide) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t lfull[LSTAGES], lempty[LSTAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* lring = base + 8 * EB * 4096;
  if (threadIdx.x == 0) {
    for (int i = 0; i < LSTAGES; ++i) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  uint32_t acc_x = 0;
  if (loads && warp == 0 && lane == 0) {  // producer: the operand boxes of every tile (2 k-blocks each)
    const uint64_t hl = policy_evict_last();
    uint32_t st = 0, ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t / (TKV / TNC)) * TMR % TQ, n0 = (t % (TKV / TNC)) * TNC;
      for (int kb = 0; kb < 2; ++kb) {
        mbar_wait(&lempty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&lfull[st], loads == 1 ? LSTAGE_BYTES : LSTAGE_BYTES / 2);
        if (loads == 1) tma_load_2d(lring + st * LSTAGE_BYTES, &a_map, &lfull[st], kb * 64, m0, hl);
        tma_load_2d(lring + st * LSTAGE_BYTES + LSTAGE_BYTES / 2, &b_map, &lfull[st], kb * 64, n0 % TKV, hl);
        if (++st == LSTAGES) st = 0, ph ^= 1u;
      }
    }
  } else if (loads && warp == 1 && lane == 0) {  // consumer: frees each stage as soon as it landed
    uint32_t st = 0, ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int kb = 0; kb < 2; ++kb) {
        mbar_wait(&lfull[st], ph);
        mbar_arrive(&lempty[st]);
        if (++st == LSTAGES) st = 0, ph ^= 1u;
      }
    }
  }
  if (warp >= 2) {
    const int quarter = warp & 3, half = (warp - 2) / 4, row = quarter * 32 + lane;
    uint8_t* buf = base + (warp - 2) * (EB * 4096);
    const uint64_t hint = hint_kind == 0 ? policy_evict_first() : hint_kind == 1 ? policy_evict_normal()
                                                                                 : policy_evict_last();
    uint32_t bi = 0, it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      // order 0: row-major tiles (a wave covers long row segments); 1: column-major (a wave covers
      // one 256-column strip of many row blocks); 2: row-major in 8-tile-row bands
      int m0, n0;
      if (order == 0) {
        m0 = (t / (TKV / TNC)) * TMR % TQ, n0 = (t % (TKV / TNC)) * TNC;
      } else if (order == 1) {
        m0 = (t % (TQ / TMR)) * TMR, n0 = (t / (TQ / TMR)) * TNC % TKV;
      } else {
        const int band = t / (8 * (TKV / TNC)), in = t % (8 * (TKV / TNC));
        m0 = (band * 8 + in % 8) * TMR % TQ, n0 = (in / 8) * TNC;
      }
      const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + (it & 1u) * 256;
      for (int ci = 0; ci < 2; ++ci) {
        const int c64 = wide ? half * 2 + ci : half + 2 * ci;
        if ((mode == M_TMA || mode == M_FULL) && (!wide || ci == 0)) {
          if (lane == 0) {
            if (wide) tma_store_wait_read<0>();  // wide: one 8 KB store (2 buffers) in flight per warp
            else tma_store_wait_read<EB - 1>();
          }
          __syncwarp();
        }
        if (wide) bi = ci;
        for (int h = 0; h < 2; ++h) {
          uint32_t v[32];
          if (mode == M_LDTM || mode == M_LDSTS || mode == M_FULL) {
            tmem_ld_32x32b_x32(taddr + c64 * 64 + 32 * h, v);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = uint32_t(i * 0x3f800000u + row + it);
          }
          if (mode == M_LDTM) {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc_x ^= v[i];
            continue;
          }
          uint4 w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w[q].x = pack_bf16x2(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
            w[q].y = pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
            w[q].z = pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
            w[q].w = pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(buf + bi * 4096 + swz128(lane, 4 * h + q)) = w[q];
        }
        if ((mode == M_TMA || mode == M_FULL) && wide) {
          if (ci == 1) {
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;"
                  ::"l"(reinterpret_cast<uint64_t>(&out3_map)), "r"(smem_addr(buf)), "r"(0), "r"(m0 + quarter * 32),
                  "r"((n0 + half * 128) / 64), "l"(hint)
                  : "memory");
              tma_store_commit();
            }
          }
        } else if (mode == M_TMA || mode == M_FULL) {
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            if (hint_kind == 3)
              tma_store_2d(&out_map, buf + bi * 4096, n0 + c64 * 64, m0 + quarter * 32);
            else
              tma_store_2d_hint(&out_map, buf + bi * 4096, n0 + c64 * 64, m0 + quarter * 32, hint);
            tma_store_commit();
          }
          bi = bi + 1 == EB ? 0 : bi + 1;
        } else {
          __syncwarp();
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
  }
  if (acc_x == 0x12345678u) sink[threadIdx.x] = acc_x;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

int main() {
  void* out;
  const size_t bytes = size_t(TQ) * TKV * 2;
  CK(cudaMalloc(&out, bytes));
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4096));
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(TKV), cuuint64_t(TQ)};
  cuuint64_t strides[1] = {cuuint64_t(TKV) * 2};
  cuuint32_t box[2] = {64, 32};
  cuuint32_t estr[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    std::printf("tensor map encode failed\n");
    return 1;
  }
  const int smem = 1024 + 8 * EB * 4096 + LSTAGES * LSTAGE_BYTES;
  void *qa, *kb;
  CK(cudaMalloc(&qa, size_t(TQ) * 128 * 2));
  CK(cudaMalloc(&kb, size_t(TKV) * 128 * 2));
  CUtensorMap amap, bmap, map3;
  {  // the output as [TKV / 64 column chunks][TQ rows][64 cols]: a (64, 32, 2) box = 32 rows x 128 columns
    cuuint64_t d3[3] = {64, cuuint64_t(TQ), cuuint64_t(TKV / 64)};
    cuuint64_t s3[2] = {cuuint64_t(TKV) * 2, 128};
    cuuint32_t b3[3] = {64, 32, 2};
    cuuint32_t e3[3] = {1, 1, 1};
    if (cuTensorMapEncodeTiled(&map3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, out, d3, s3, b3, e3,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      std::printf("3d map encode failed\n");
      return 1;
    }
  }
  for (int i = 0; i < 2; ++i) {
    cuuint64_t d2[2] = {128, cuuint64_t(i ? TKV : TQ)};
    cuuint64_t s2[1] = {256};
    cuuint32_t b2[2] = {64, 128};
    if (cuTensorMapEncodeTiled(i ? &bmap : &amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, i ? kb : qa, d2, s2, b2, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      std::printf("operand map encode failed\n");
      return 1;
    }
  }
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int tiles = (TQ / TMR) * (TKV / TNC);
  const char* names[] = {"ldtm", "sts", "tma", "ldsts", "full"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* hints[] = {"evict_first", "evict_normal", "evict_last", "none"};
  struct V { int mode, hint, order, loads, wide; };
  std::vector<V> vs;
  for (int w = 0; w < 2; ++w)
    for (int l = 0; l < 3; ++l) vs.push_back({M_FULL, 0, 0, l, w});
  vs.push_back({M_TMA, 0, 0, 1, 0});
  vs.push_back({M_TMA, 0, 0, 1, 1});
  for (int round = 0; round < 2; ++round) {
    for (const V& v : vs) {
      const int mode = v.mode;
      std::vector<float> ms;
      for (int r = 0; r < 8; ++r) {
        cudaEventRecord(a);
        probe<<<sms, NT, smem>>>(map, amap, bmap, mode, tiles, sink, v.hint, v.order, v.loads, map3, v.wide);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float t;
        cudaEventElapsedTime(&t, a, b);
        ms.push_back(t);
      }
      CK(cudaGetLastError());
      std::sort(ms.begin(), ms.end());
      const double med = ms[ms.size() / 2] * 1e-3;
      // bytes of bf16 output the epilogue produces (ldtm: 2x that read from TMEM)
      std::printf("{\"round\": %d, \"mode\": \"%s\", \"hint\": \"%s\", \"order\": %d, \"loads\": %d, "
                  "\"wide\": %d, \"us_median\": %.1f, \"us_best\": %.1f, \"out_TBps\": %.3f}\n",
                  round, names[mode], hints[v.hint], v.order, v.loads, v.wide, med * 1e6, ms[0] * 1e3,
                  bytes / med / 1e12);
    }
  }
  return 0;
}

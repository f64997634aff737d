// Persistent, flag-gated tcgen05 tile kernel: the compute half of every FiCCO schedule.
//
// One CTA per SM walks a host-lowered tile list (ficco_tile) in order; tile t
// goes to CTA t mod gridDim.x. With CG = 2 (cta_group::2) the CTAs of a
// cluster pair process tiles 2p (leader, even CTA) and 2p+1 together as one
// 256 x TN MMA tile: each CTA TMA-loads its own 128 A rows and half of the B
// rows, the leader issues tcgen05.mma.cta_group::2 over both CTAs' shared
// memory, and each CTA's epilogue drains its own TMEM half. The two halves
// may come from different (non-adjacent) row fragments — e.g. fine chunks of
// two different peers — since A rows are loaded per CTA. Warp roles (192 threads):
//   warp 0      TMA producer: waits the tile's readiness flag(s) (written by
//               copy-engine stream memops or by peers), then streams 128x64 A
//               and 256x64 B boxes (128B swizzle) into a STAGES-deep ring.
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               (kind::f16, M=128 N=256 K=16) into one of two TMEM accumulators
//               (2 x 256 fp32 columns) so the epilogue of tile i overlaps the
//               MMAs of tile i+1.
//   warps 2-5   epilogue: tcgen05.ld 32x32b (one accumulator row per thread),
//               scale / reduce, bf16 pack, masked 16-byte stores at
//               (c_row, c_col) — the reference's ScatterSpec folded into the
//               store addressing (planner.py:262-271).
//
// A schedule kind is nothing but a tile ORDER plus a DEPENDENCY SET:
//   uniform_fused_1d  step-major tiles, each gated on its round's flag
//   hetero_*_1d       local-shard tiles first (no wait), then rounds
//   uniform_fused_2d  output-stationary tiles, k-block kb gated on round kb/kseg
//                     (TMEM-resident accumulation replaces the chained additive
//                     GEMMs of planner.py:368-383)
//   shard_overlap     shard-major tiles gated on the ring step's flag
#pragma once

#include "../../include/ficco.h"
#include "sm100_primitives.cuh"

namespace ficco {

constexpr int BM = 128;      // rows per CTA (UMMA M = 128 * CG)
constexpr int BN_MAX = 256;  // widest tile (UMMA N <= 256); per-plan tile width TN in {128,...,256}
constexpr int BK = 64;       // 64 bf16 = 128 B = one swizzle row
constexpr int UMMA_K = 16;
constexpr int A_STAGE = BM * BK * 2;  // 16 KiB
constexpr int EPI_WARPS = 8;   // two epilogue warps per TMEM lane quarter (alternating 32-column chunks)
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr int NUM_THREADS = 64 + EPI_THREADS;
// Register cap. The persistent kernel occupies every SM for the whole op while the
// copy program runs beside it; same-device strided copies (the virtual peers' pulls,
// local publishes) may be executed by the driver as small SM copy kernels, which must
// still fit next to one tile CTA. At 168 registers/thread the co-resident copy CTA no
// longer fits and the copy program stalls behind the kernel that waits on it.
constexpr int MAX_REGS = 128;
constexpr int COPY_RESERVE_REGS = 65536 - MAX_REGS * NUM_THREADS;
constexpr uint32_t TMEM_COLS = 512;  // two accumulators of up to 256 fp32 columns
constexpr int MAX_RECV = 15;
constexpr int MAX_PEERS = MAX_RECV + 1;
constexpr int SMEM_LIMIT = 226 * 1024;  // leaves room for the static smem (seen-flag bitset)
// Epilogue output staging: per epilogue warp EB buffers of one 32-row x 64-column bf16
// box (128 B rows, TMA SWIZZLE_128B layout: full-line writes), stored with
// cp.async.bulk.tensor; a trailing 32-column chunk uses a 32 x 32 box (SWIZZLE_64B).
// EB staging buffers per warp keep EB bulk stores in flight: 1 for long-K (MMA-bound) tile
// programs, where smem is better spent on pipeline stages, 3 for short-K programs (C4's
// d = 128), whose tiles are store-bound (see lowering.epi_bufs_for / ficco.cu epi_bufs_for).
constexpr int EPI_BUF_BYTES = 32 * 128;

// Per (tile width, CTA group) configuration: as many pipeline stages as fit.
template <int TN, int CG, int EB = 1>
struct TileCfg {
  static_assert(TN % 32 == 0 && TN >= 64 && TN <= 256, "tile width");
  static_assert(CG == 1 || CG == 2, "cta group");
  static constexpr int B_ROWS = TN / CG;  // B rows loaded by each CTA
  static constexpr int B_STAGE = B_ROWS * BK * 2;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static_assert(EB >= 1 && EB <= 4, "epilogue staging buffers");
  static constexpr int EPI_STAGE_BYTES = EB * EPI_BUF_BYTES * EPI_WARPS;  // TMA-store staging
  static constexpr int MAX_STAGES = (SMEM_LIMIT - 1024 - 256 - EPI_STAGE_BYTES) / STAGE;
  static constexpr int STAGES = MAX_STAGES > 8 ? 8 : MAX_STAGES;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE + EPI_STAGE_BYTES + 256;
  // REDUCE tiles: per peer, RKB extra k-blocks D[:, 64i:64i+64] += P_j[:, 64i:64i+64] * I_64
  static constexpr int RKB = (TN + 63) / 64;
  static constexpr int IDENT_ROWS = 64 / CG;  // identity rows (UMMA N split) loaded by each CTA
  static constexpr int RED_STAGE = A_STAGE + IDENT_ROWS * BK * 2;
};

struct alignas(64) TileParams {
  CUtensorMap tmap_a;
  CUtensorMap tmap_b;
  CUtensorMap tmap_a2;  // alternate sources (e.g. the caller's local shard, read in place)
  CUtensorMap tmap_b2;
  CUtensorMap tmap_out;     // 64 x 32 store boxes, SWIZZLE_128B (STORE / REDUCE destination)
  CUtensorMap tmap_part;    // same for the STORE_SIGNAL destination
  CUtensorMap tmap_out32;   // 32 x 32 boxes, SWIZZLE_64B (trailing 32-column chunks)
  CUtensorMap tmap_part32;
  CUtensorMap tmap_recv;    // receive slots as one [n_recv * recv_rows, N] matrix, 128 x 64 boxes (A layout)
  CUtensorMap tmap_ident;   // 64 x 64 bf16 identity, (64 / CG) x 64 boxes (B layout)
  // STORE_REMOTE (comm_agent = core GEMM -> RS): per owner rank q, this rank's receive slot in q's
  // workspace (peer memory), 64- and 32-column store boxes, and q's flag block of this run
  CUtensorMap tmap_rem[MAX_PEERS];
  CUtensorMap tmap_rem32[MAX_PEERS];
  __nv_bfloat16* rem[MAX_PEERS];
  uint32_t* rem_flags[MAX_PEERS];
  int64_t ld_rem;
  int has_rem_map;
  int go_flag;             // STORE_REMOTE stores wait for local flag[go_flag] (<= 0: none)
  int go_all;              // STORE_SIGNAL stores wait for it too (nvls: peers read the partials in place)
  uint32_t rs_target;      // REDUCE waits its peers' flags >= rs_target
  int has_out_map;
  int has_part_map;
  const ficco_tile* tiles;
  int num_tiles;
  int num_kb;
  __nv_bfloat16* out;      // STORE / REDUCE destination
  __nv_bfloat16* part;     // STORE_SIGNAL destination
  int64_t ld_out;
  int64_t ld_part;
  const __nv_bfloat16* recv[MAX_RECV];
  int64_t ld_recv;
  int n_recv;
  int rs_flag0;
  int reduce_mma;          // REDUCE tiles fold the peers' partials in with identity MMAs (else epilogue loads;
                           // 2: boxes streamed through the ring without the MMAs, timing experiments only)
  int recv_rows;           // rows per receive slot in tmap_recv (slot j starts at row j * recv_rows)
  int b_resident;          // short-K programs: a CTA's B rows stay in smem while consecutive tiles share them
                           // (b_row, b_src): only A is streamed through the ring (halves the L2->SM bytes
                           // of C4's store-bound tiles). Requires num_kb <= STAGES and no REDUCE tiles.
  int a_evict_last;        // FICCO_HINT_A_EVICT_LAST
  int b_evict_first;       // FICCO_HINT_B_EVICT_FIRST (1; 2: evict_normal, FICCO_B_HINT experiments)
  int part_hint;           // L2 policy of STORE_SIGNAL (to-be-pushed) stores: 0 evict_first, 1 normal, 2 last
  int epi_fast;            // full 64-column chunks take the straight-line epilogue path (FICCO_EPI_FAST=0: off)
  int epi_x64;             // the fast path reads its 64 columns with one tcgen05.ld .x64 (FICCO_EPI_X64=1)
  int out_plain;           // STORE / REDUCE output boxes stored without an L2 policy (store-bound programs:
                           // +10 % HBM write rate over evict_first, tools/epi_probe.cu)
  uint32_t* flags;         // local flag block of this run's parity
  uint32_t* counters;      // local tile counters
  uint32_t* abort_word;
  uint32_t* abort_host;    // host-mapped mirror of abort_word (ficco_plan_run refuses a poisoned communicator)
  uint32_t epoch;          // value a flag must reach (1: one-shot flags)
  unsigned long long timeout_ns;  // flag waits abort after this long (FICCO_FLAG_TIMEOUT_S, default 30 s)
  float alpha;
  // optional timeline (ns, %globaltimer): [0, gridDim) CTA start; then per tile
  // {loads may start (flags satisfied), accumulator stored}
  unsigned long long* trace;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Poll a flag written by another agent (copy engine, peer GPU) until it reaches
// `epoch` (wrap-safe) with acquire loads (a sys-scope fence per flag would cost
// microseconds; the acquire load itself orders the following reads). After
// `timeout_ns` of waiting (%globaltimer; TileParams.timeout_ns) raise the abort word
// and give up so the kernel drains instead of hanging the device.
__device__ __forceinline__ void wait_flag(const uint32_t* f, uint32_t epoch, uint32_t* abort_word,
                                          unsigned long long timeout_ns, uint32_t* abort_host) {
  uint32_t spins = 0;
  unsigned long long t0 = 0;
  while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
    if ((++spins & 1023u) == 0) {
      const unsigned long long now = globaltimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns) {
        // non-zero; the low bits name the word that never arrived (ficco_comm_check reports it)
        atomicExch(abort_word, 0x80000000u | (uint32_t(reinterpret_cast<uintptr_t>(f)) & 0x7fffffffu));
        if (abort_host) {
          *reinterpret_cast<volatile uint32_t*>(abort_host) = 1u;
          __threadfence_system();
        }
        break;
      }
      if (*reinterpret_cast<volatile uint32_t*>(abort_word)) break;
    }
    __nanosleep(64);
  }
  // make the copy-engine-written bytes visible to the async (TMA) proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One-shot flags never go back to 0 within a run, so the (single-thread) producer
// remembers which ones it has already seen: a tile gated by G-1 round flags costs
// G-1 global polls only the first time, then a bit test per flag.
constexpr int SEEN_WORDS = FICCO_FLAG_BLOCK / 32;

__device__ __forceinline__ void wait_flag_cached(uint32_t* seen, const uint32_t* flags, int idx, uint32_t epoch,
                                                 uint32_t* abort_word, unsigned long long timeout_ns,
                                                 uint32_t* abort_host) {
  const uint32_t bit = 1u << (idx & 31);
  if (seen[idx >> 5] & bit) return;
  wait_flag(flags + idx, epoch, abort_word, timeout_ns, abort_host);
  seen[idx >> 5] |= bit;
}

template <int TN, int CG, int EB>
__device__ __forceinline__ void producer_loop(const TileParams& p, uint8_t* sA, uint8_t* sB, uint64_t* full,
                                              uint64_t* empty, uint32_t rank, uint32_t* seen, uint64_t* bfree) {
  using Cfg = TileCfg<TN, CG, EB>;
  const uint64_t hint_a = p.a_evict_last ? policy_evict_last() : policy_evict_first();
  const uint64_t hint_b = p.b_evict_first == 1   ? policy_evict_first()
                          : p.b_evict_first == 2 ? policy_evict_normal()
                                                 : policy_evict_last();
  const uint64_t hint_recv = policy_evict_first();  // received partials are read once (REDUCE)
  uint32_t stage = 0, phase = 0;
  int res_b_row = -1, res_b_src = -1, res_b_cols = -1;  // B rows resident in smem (b_resident mode)
  uint32_t bfree_phase = 0;
  for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
    const ficco_tile td = p.tiles[t];
    // per-tile MMA width (tile cols, a multiple of 32 <= TN): with CTA pairs each CTA supplies half of
    // the UMMA N rows, so the second CTA's B rows start cols/2 (not TN/2) past the tile's first row
    const int b_row = td.b_row + int(rank) * (CG == 2 ? td.cols / 2 : 0);
    const CUtensorMap* map_a = td.a_src ? &p.tmap_a2 : &p.tmap_a;
    const CUtensorMap* map_b = td.b_src ? &p.tmap_b2 : &p.tmap_b;
    // b_resident: (re)load B only when this tile's B rows differ from the resident ones, after the MMAs
    // of every tile that read the old rows completed (b_free, committed by the MMA issuer)
    const bool load_b =
        !p.b_resident || td.b_row != res_b_row || int(td.b_src) != res_b_src || int(td.cols) != res_b_cols;
    if (p.b_resident && load_b) {
      if (res_b_row >= 0) {
        mbar_wait(bfree, bfree_phase);
        bfree_phase ^= 1u;
      }
      res_b_row = td.b_row;
      res_b_src = td.b_src;
      res_b_cols = td.cols;
    }
    for (int kb = 0; kb < p.num_kb; ++kb) {
      if (td.flag >= 0) {
        int base = -1;
        if (td.kseg == 0) {
          if (kb == 0) base = td.flag;
        } else if (kb % td.kseg == 0) {
          base = td.flag + (kb / td.kseg) * td.kstride;
        }
        if (base >= 0) {
          // fast path: every gating flag already observed (one 64-bit window test)
          const uint32_t w0 = seen[base >> 5], w1 = (base >> 5) + 1 < SEEN_WORDS ? seen[(base >> 5) + 1] : 0u;
          const uint32_t window = uint32_t(((uint64_t(w1) << 32) | w0) >> (base & 31));
          if ((window & td.fmask) != td.fmask)
            for (uint32_t m = td.fmask; m; m &= m - 1)
              wait_flag_cached(seen, p.flags, base + (__ffs(m) - 1), p.epoch, p.abort_word, p.timeout_ns,
                               p.abort_host);
        }
      }
      if (kb == 0 && p.trace) p.trace[gridDim.x + 2 * t] = globaltimer();
      mbar_wait(&empty[stage], phase ^ 1u);
      // resident B of k-block kb lives in the B slot of stage kb (the A ring uses only the A slots)
      uint8_t* dst_b = sB + (p.b_resident ? kb : int(stage)) * Cfg::B_STAGE;
      const uint32_t bytes = load_b ? Cfg::STAGE : A_STAGE;
      if constexpr (CG == 1) {
        mbar_arrive_expect_tx(&full[stage], bytes);
        tma_load_2d(sA + stage * A_STAGE, map_a, &full[stage], kb * BK, td.a_row, hint_a);
        if (load_b) tma_load_2d(dst_b, map_b, &full[stage], kb * BK, b_row, hint_b);
      } else {
        // both CTAs' bytes complete on the leader's barrier; the leader arms it for the pair (the pair's
        // tiles share b_row, so both CTAs agree on load_b)
        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
        tma_load_2d_pair(sA + stage * A_STAGE, map_a, &full[stage], kb * BK, td.a_row, hint_a);
        if (load_b) tma_load_2d_pair(dst_b, map_b, &full[stage], kb * BK, b_row, hint_b);
      }
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (p.reduce_mma && td.mode == FICCO_EPI_REDUCE) {
      // GEMM -> RS owner tile: the peers' partial chunks (copy-engine pushed into our
      // receive slots) stream through the same ring as A operands against an identity B,
      // so the reduction rides the TMA/tensor pipeline instead of the epilogue's loads.
      for (int j = 0; j < p.n_recv; ++j)
        wait_flag_cached(seen, p.flags, p.rs_flag0 + td.chunk * p.n_recv + j, p.rs_target, p.abort_word,
                         p.timeout_ns, p.abort_host);
      for (int j = 0; j < p.n_recv; ++j) {
        for (int kb = 0; kb < Cfg::RKB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          const int rrow = j * p.recv_rows + td.recv_row;
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full[stage], Cfg::RED_STAGE);
            tma_load_2d(sA + stage * A_STAGE, &p.tmap_recv, &full[stage], td.c_col + kb * 64, rrow, hint_recv);
            tma_load_2d(sB + stage * Cfg::B_STAGE, &p.tmap_ident, &full[stage], 0, 0, hint_b);
          } else {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::RED_STAGE);
            tma_load_2d_pair(sA + stage * A_STAGE, &p.tmap_recv, &full[stage], td.c_col + kb * 64, rrow, hint_recv);
            tma_load_2d_pair(sB + stage * Cfg::B_STAGE, &p.tmap_ident, &full[stage], 0,
                             int(rank) * Cfg::IDENT_ROWS, hint_b);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  }
}

template <int TN, int CG, int EB>
__device__ __forceinline__ void mma_loop(const TileParams& p, uint8_t* sA, uint8_t* sB, uint64_t* full,
                                         uint64_t* empty, uint64_t* tfull, uint64_t* tempty, uint32_t tmem,
                                         uint64_t* bfree) {
  using Cfg = TileCfg<TN, CG, EB>;
  constexpr uint32_t idesc64 = make_idesc_bf16(BM * CG, 64);
  uint32_t stage = 0, phase = 0, it = 0;
  for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
    // UMMA N = the tile's own width (per-chunk tile shapes; cols % 32 == 0 and <= TN, ficco_plan_create)
    const uint32_t idesc = make_idesc_bf16(BM * CG, p.tiles[t].cols);
    const uint32_t acc = it & 1u;
    mbar_wait(&tempty[acc], ((it >> 1) & 1u) ^ 1u);
    tc_fence_after();
    const uint32_t d = tmem + acc * BN_MAX;
    for (int kb = 0; kb < p.num_kb; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint64_t ad = make_sdesc_sw128(smem_addr(sA + stage * A_STAGE));
      const uint64_t bd = make_sdesc_sw128(smem_addr(sB + (p.b_resident ? kb : int(stage)) * Cfg::B_STAGE));
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k) {
        // +32 bytes per K step inside the 128B swizzle row (>>4 in the descriptor)
        if constexpr (CG == 1)
          umma_bf16(d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
        else
          umma_bf16_pair(d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
      }
      if constexpr (CG == 1)
        umma_commit(&empty[stage]);  // smem slot free once these MMAs retire
      else
        umma_commit_pair(&empty[stage]);  // ... in both CTAs of the pair
      if (++stage == Cfg::STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (p.reduce_mma && p.tiles[t].mode == FICCO_EPI_REDUCE) {
      // D[:, 64i:64i+64] += P_j[:, 64i:64i+64] x I_64 for every peer j (rank-ascending)
      for (int j = 0; j < p.n_recv * Cfg::RKB; ++j) {
        const uint32_t col = uint32_t(j % Cfg::RKB) * 64u;
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = make_sdesc_sw128(smem_addr(sA + stage * A_STAGE));
        const uint64_t bd = make_sdesc_sw128(smem_addr(sB + stage * Cfg::B_STAGE));
#pragma unroll
        for (int k = 0; k < BK / UMMA_K && p.reduce_mma == 1; ++k) {  // 2: timing only, loads without adds
          if constexpr (CG == 1)
            umma_bf16(d + col, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc64, 1u);
          else
            umma_bf16_pair(d + col, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc64, 1u);
        }
        if constexpr (CG == 1)
          umma_commit(&empty[stage]);
        else
          umma_commit_pair(&empty[stage]);
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    if constexpr (CG == 1)
      umma_commit(&tfull[acc]);  // accumulator complete
    else
      umma_commit_pair(&tfull[acc]);
    if (p.b_resident) {
      // the resident B rows are free once this tile's MMAs retire, if the CTA's next tile reads other rows
      const int nt = t + int(gridDim.x);
      if (nt < p.num_tiles && (p.tiles[nt].b_row != p.tiles[t].b_row || p.tiles[nt].b_src != p.tiles[t].b_src ||
                               p.tiles[nt].cols != p.tiles[t].cols)) {
        if constexpr (CG == 1)
          umma_commit(bfree);
        else
          umma_commit_pair(bfree);
      }
    }
  }
}

// Byte offset of 16-byte chunk j of row t in a TMA SWIZZLE_64B box (64 B rows, Swizzle<2,4,3>)
// and in a SWIZZLE_128B box (128 B rows, Swizzle<3,4,3>).
__device__ __forceinline__ uint32_t swz64(uint32_t t, uint32_t j) { return t * 64u + ((j ^ ((t >> 1) & 3u)) << 4); }
__device__ __forceinline__ uint32_t swz128(uint32_t t, uint32_t j) { return t * 128u + ((j ^ (t & 7u)) << 4); }

// TMEM columns [col, col+32) of this thread's row -> scaled fp32 (+ peers' partials) -> 4 packed uint4.
__device__ __forceinline__ void epi_chunk(const TileParams& p, const ficco_tile& td, uint32_t taddr, int col,
                                          float scale, bool reduce_row, int row, uint4 (&w)[4]) {
  uint32_t v[32];
  tmem_ld_32x32b_x32(taddr + col, v);
  tmem_ld_wait();
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
  if (scale != 1.0f) {
    // packed fp32x2 multiplies (FMUL2): short-K epilogues are issue-bound, the scale is half their ALU work
    const uint64_t s2 = f32x2(scale, scale);
#pragma unroll
    for (int i = 0; i < 32; i += 2) fmul2(f[i], f[i + 1], s2);
  }
  if (reduce_row) {
    // rank-ascending sum of the peers' partial chunks; the next peer's 64 bytes are in
    // flight while the current ones are added (the loads are latency-, not bandwidth-bound)
    const int64_t roff = int64_t(td.recv_row + row) * p.ld_recv + td.c_col + col;
    uint4 cur[4], nxt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) cur[q] = __ldcs(reinterpret_cast<const uint4*>(p.recv[0] + roff) + q);
    for (int j = 0; j < p.n_recv; ++j) {
      if (j + 1 < p.n_recv) {
#pragma unroll
        for (int q = 0; q < 4; ++q) nxt[q] = __ldcs(reinterpret_cast<const uint4*>(p.recv[j + 1] + roff) + q);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&cur[q]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 x = __bfloat1622float2(h[e]);
          f[q * 8 + 2 * e] += x.x;
          f[q * 8 + 2 * e + 1] += x.y;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w[q].x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
    w[q].y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
    w[q].z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
    w[q].w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
  }
}

template <int TN, int CG, int EB>
__device__ __forceinline__ void epilogue_loop(const TileParams& p, uint64_t* tfull, uint64_t* tempty,
                                              uint32_t tmem, uint8_t* stage_smem) {
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const int quarter = warp & 3;           // TMEM lane quarter this warp may access
  const int half = (warp - 2) / 4;        // which alternate 64-column chunks this warp drains
  const int row = quarter * 32 + lane;
  const uint64_t hint_out = policy_evict_first();  // results stream out; keep operands resident in L2
  // partial chunks are read back by the push copies right after their unit completes
  const uint64_t hint_part = p.part_hint == 2 ? policy_evict_last()
                             : p.part_hint == 1 ? policy_evict_normal() : hint_out;
  uint8_t* buf = stage_smem + (warp - 2) * (EB * EPI_BUF_BYTES);
  uint32_t bi = 0;  // staging buffer of the next bulk store (round robin over EB)
  bool go_seen = false;
  uint32_t it = 0;
  for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
    const ficco_tile td = p.tiles[t];
    const uint32_t acc = it & 1u;
    const bool epi_reduce = td.mode == FICCO_EPI_REDUCE && !p.reduce_mma;  // partials added from global
    if (epi_reduce) {
      // peers' partial chunks must have landed in our receive slots
      if (threadIdx.x == 64) {
        for (int j = 0; j < p.n_recv; ++j)
          wait_flag(p.flags + p.rs_flag0 + td.chunk * p.n_recv + j, p.rs_target, p.abort_word, p.timeout_ns,
                    p.abort_host);
      }
      named_bar_sync(1, EPI_THREADS);
    }
    mbar_wait(&tfull[acc], (it >> 1) & 1u);
    tc_fence_after();
    const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + acc * BN_MAX;
    const bool row_ok = row < td.rows;
    const bool signal = td.mode == FICCO_EPI_STORE_SIGNAL;
    const bool remote = td.mode == FICCO_EPI_STORE_REMOTE;  // td.chunk = owner rank
    const bool reduce_row = epi_reduce && row_ok;
    if ((remote || (signal && p.go_all)) && !go_seen) {
      // the owners' receive slots are free once the DONE barrier of this run passed
      if (p.go_flag > 0 && lane == 0)
        wait_flag(p.flags + p.go_flag, p.epoch, p.abort_word, p.timeout_ns, p.abort_host);
      __syncwarp();
      go_seen = true;
    }
    // whole 32-row warp boxes go out through TMA stores; ragged rows use direct stores
    const int warp_rows = td.rows - quarter * 32;
    const bool tma = warp_rows >= 32 && (remote ? p.has_rem_map : signal ? p.has_part_map : p.has_out_map);
    const CUtensorMap* map64 = remote ? &p.tmap_rem[td.chunk] : signal ? &p.tmap_part : &p.tmap_out;
    const CUtensorMap* map32 = remote ? &p.tmap_rem32[td.chunk] : signal ? &p.tmap_part32 : &p.tmap_out32;
    __nv_bfloat16* dst = remote ? p.rem[td.chunk] + int64_t(td.c_row + row) * p.ld_rem + td.c_col
                         : signal ? p.part + int64_t(td.c_row + row) * p.ld_part + td.c_col
                                  : p.out + int64_t(td.c_row + row) * p.ld_out + td.c_col;
    const float scale = td.mode == FICCO_EPI_STORE ? p.alpha : 1.0f;
#pragma unroll 1
    for (int c64 = half; c64 * 64 < TN; c64 += 2) {
      const int col = c64 * 64;
      const bool live1 = col + 64 <= TN && col + 32 < td.cols;  // warp-uniform
      if (col >= td.cols) continue;
      if (tma) {
        // the buffer about to be refilled was handed to the store issued EB stores ago
        if (lane == 0) tma_store_wait_read<EB - 1>();
        __syncwarp();
      }
      if (p.epi_fast && tma && !reduce_row && col + 64 <= td.cols) {
        // fast path (every full 64-column chunk without epilogue reduction): both 32-column TMEM loads
        // in flight before one wait, scale, pack, eight 16-byte swizzled st.shared, one TMA store
        uint32_t v[64];
        uint32_t* v0 = v;
        uint32_t* v1 = v + 32;
        if (p.epi_x64) {
          tmem_ld_32x32b_x64(taddr + col, v);
        } else {
          tmem_ld_32x32b_x32(taddr + col, *reinterpret_cast<uint32_t(*)[32]>(v0));
          tmem_ld_32x32b_x32(taddr + col + 32, *reinterpret_cast<uint32_t(*)[32]>(v1));
        }
        tmem_ld_wait();
        const uint32_t srow = smem_addr(buf + bi * EPI_BUF_BYTES) + uint32_t(lane) * 128u;
        const uint32_t l7 = uint32_t(lane) & 7u;
        if (scale != 1.0f) {
          const uint64_t s2 = f32x2(scale, scale);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float x0 = __uint_as_float(v0[i]), y0 = __uint_as_float(v0[i + 1]);
            float x1 = __uint_as_float(v1[i]), y1 = __uint_as_float(v1[i + 1]);
            fmul2(x0, y0, s2);
            fmul2(x1, y1, s2);
            v0[i] = __float_as_uint(x0), v0[i + 1] = __float_as_uint(y0);
            v1[i] = __float_as_uint(x1), v1[i + 1] = __float_as_uint(y1);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t* f = v0 + 8 * j;
          st_shared_v4(srow + ((uint32_t(j) ^ l7) << 4),
                       pack_bf16x2(__uint_as_float(f[0]), __uint_as_float(f[1])),
                       pack_bf16x2(__uint_as_float(f[2]), __uint_as_float(f[3])),
                       pack_bf16x2(__uint_as_float(f[4]), __uint_as_float(f[5])),
                       pack_bf16x2(__uint_as_float(f[6]), __uint_as_float(f[7])));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t* f = v1 + 8 * j;
          st_shared_v4(srow + ((uint32_t(j + 4) ^ l7) << 4),
                       pack_bf16x2(__uint_as_float(f[0]), __uint_as_float(f[1])),
                       pack_bf16x2(__uint_as_float(f[2]), __uint_as_float(f[3])),
                       pack_bf16x2(__uint_as_float(f[4]), __uint_as_float(f[5])),
                       pack_bf16x2(__uint_as_float(f[6]), __uint_as_float(f[7])));
        }
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          if (p.out_plain && !signal && !remote)
            tma_store_2d(map64, buf + bi * EPI_BUF_BYTES, td.c_col + col, td.c_row + quarter * 32);
          else
            tma_store_2d_hint(map64, buf + bi * EPI_BUF_BYTES, td.c_col + col, td.c_row + quarter * 32,
                              signal ? hint_part : hint_out);
          tma_store_commit();
        }
        bi = bi + 1 == EB ? 0 : bi + 1;
        continue;
      }
      // the two 32-column halves one after the other: one half's values live at a time
#pragma unroll 1
      for (int h = 0; h < (live1 ? 2 : 1); ++h) {
        uint4 w[4];
        epi_chunk(p, td, taddr, col + 32 * h, scale, reduce_row, row, w);
        if (tma) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(buf + bi * EPI_BUF_BYTES + (live1 ? swz128(lane, 4 * h + q) : swz64(lane, q))) =
                w[q];
        } else if (row_ok) {
          uint4* o = reinterpret_cast<uint4*>(dst + col + 32 * h);
#pragma unroll
          for (int q = 0; q < 4; ++q) o[q] = w[q];
        }
      }
      if (tma) {
        fence_async_shared();
        __syncwarp();
        if (lane == 0) {
          if (p.out_plain && !signal && !remote)
            tma_store_2d(live1 ? map64 : map32, buf + bi * EPI_BUF_BYTES, td.c_col + col, td.c_row + quarter * 32);
          else
            tma_store_2d_hint(live1 ? map64 : map32, buf + bi * EPI_BUF_BYTES, td.c_col + col,
                              td.c_row + quarter * 32, signal ? hint_part : hint_out);
          tma_store_commit();
        }
        bi = bi + 1 == EB ? 0 : bi + 1;
      }
    }
    tc_fence_before();
    if constexpr (CG == 1)
      mbar_arrive(&tempty[acc]);
    else
      mbar_arrive_leader(&tempty[acc]);  // the leader's MMA reuses the pair's accumulator
    if (p.trace && threadIdx.x == 64) p.trace[gridDim.x + 2 * t + 1] = globaltimer();
    if (signal || remote) {
      if (lane == 0) tma_store_wait_all<0>();  // this warp's bulk stores are complete
      named_bar_sync(1, EPI_THREADS);          // every row of the tile is stored
      if (threadIdx.x == 64) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy (TMA) writes before the release
        __threadfence_system();
        red_release_add(remote ? p.rem_flags[td.chunk] + td.recv_row : p.counters + td.chunk, 1u);
      }
    }
  }
  if (lane == 0) tma_store_wait_all<0>();  // staging smem must outlive the bulk stores
}

template <int TN, int CG, int EB>
__global__ void __maxnreg__(MAX_REGS) tile_gemm_kernel(const __grid_constant__ TileParams p) {
  using Cfg = TileCfg<TN, CG, EB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + Cfg::STAGES * A_STAGE;
  uint8_t* sEpi = sB + Cfg::STAGES * Cfg::B_STAGE;  // 1024-aligned (stage sizes are multiples of 1 KiB)
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + Cfg::EPI_STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfree = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfree + 1);
  __shared__ uint32_t seen_flags[SEEN_WORDS];  // producer's record of flags already observed set

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x] = globaltimer();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.tmap_a);
    tma_prefetch_desc(&p.tmap_b);
    tma_prefetch_desc(&p.tmap_a2);
    tma_prefetch_desc(&p.tmap_b2);
    if (p.has_out_map) {
      tma_prefetch_desc(&p.tmap_out);
      tma_prefetch_desc(&p.tmap_out32);
    }
    if (p.has_part_map) {
      tma_prefetch_desc(&p.tmap_part);
      tma_prefetch_desc(&p.tmap_part32);
    }
    if (p.reduce_mma) {
      tma_prefetch_desc(&p.tmap_recv);
      tma_prefetch_desc(&p.tmap_ident);
    }
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_THREADS * CG);
    }
    mbar_init(bfree, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 1)
      tmem_alloc(tmem_slot, TMEM_COLS);
    else
      tmem_alloc_pair(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 1)
    __syncthreads();
  else
    cluster_sync();  // peer barriers initialised before any remote arrive / TMA complete_tx
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < SEEN_WORDS; ++i) seen_flags[i] = 0;
      producer_loop<TN, CG, EB>(p, sA, sB, full, empty, rank, seen_flags, bfree);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) mma_loop<TN, CG, EB>(p, sA, sB, full, empty, tfull, tempty, tmem, bfree);
  } else {
    epilogue_loop<TN, CG, EB>(p, tfull, tempty, tmem, sEpi);
  }

  tc_fence_before();
  if constexpr (CG == 1)
    __syncthreads();
  else
    cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (CG == 1)
      tmem_dealloc(tmem, TMEM_COLS);
    else
      tmem_dealloc_pair(tmem, TMEM_COLS);
  }
}

// (tile width, CTA group) instantiations for the per-plan choice (see lowering.choose_tile_n).
#define FICCO_FOR_EACH_CFG(X)                                                                        \
  X(128, 1, 1) X(160, 1, 1) X(192, 1, 1) X(224, 1, 1) X(256, 1, 1) X(128, 2, 1) X(160, 2, 1) X(192, 2, 1) \
  X(224, 2, 1) X(256, 2, 1) X(128, 1, 3) X(160, 1, 3) X(192, 1, 3) X(224, 1, 3) X(256, 1, 3) X(128, 2, 3) \
  X(160, 2, 3) X(192, 2, 3) X(224, 2, 3) X(256, 2, 3)

}  // namespace ficco

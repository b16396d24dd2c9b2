// RRS fused grouped GEMM on tcgen05, sm_100a.
//
//   P_g[t][n] = sum_{j' in group g} Xq8[t][j'] * Wq8[n][j']          (fig:framework (3) P:103)
//   Y[t][n]   = out_scale * alpha_t * beta_n * sum_g s_g * f32(P_g)   ("the runtime smoothing scales are
//                                                                     applied to the dequantized interim
//                                                                     result"; R14, R15)
//
// Design: persistent, one CTA per SM, 448 threads = 14 warps (<= 4 per SM sub-partition,
// so 128 registers per thread).  kCta = 2 (T > 128): CTA pairs (clusters of 2) run tcgen05 with
// cta_group::2, M = 256 (128 rows per CTA), N = 240: each CTA loads its own 128 X rows and HALF of the 240
// W rows of a group, so a CTA moves 31 KiB per 128-deep group instead of 46 KiB -- the kernel is bound
// by L2->SM bandwidth otherwise.  kCta = 1 (decode-sized T): M = 128 per CTA.
//   warp 0      TMA producer: X tile + W tile per group into a STAGES-deep SMEM ring (SWIZZLE_128B: one
//               128-code group is exactly one 128-byte swizzle row).  In a pair, both CTAs' loads
//               complete on the leader's mbarrier (cp.async.bulk.tensor .cta_group::2);
//   warp 1      TMEM allocator; in the leader, the single-thread tcgen05.mma.kind::i8 issuer (K=32, 4 per
//               group) into one of two int32 TMEM accumulators (columns [0,240), [256,496)), alternating
//               per group; commits multicast to both CTAs.  N = 240 makes the tile count of the LLaMA
//               shapes land just under a whole number of waves on 148 SMs (2048 x 4096: 144 pair tiles
//               = 1.95 waves of 74 pairs);
//   warps 2-13  promotion/epilogue (lane quadrant = warp % 4, column third = (warp-2)/4: 80 columns,
//               whose f32 accumulators stay in registers); they release a buffer on the leader's barrier.
// int8 carrier: every accumulation starts fresh (like the FP8 carrier) and the exact int32 P_g is turned into a float
// in registers with the magic-number trick -- bits(P + 0x4B400000) is the float 1.5*2^23 + P, exact because
// |P| <= 6272 < 2^22 (|sum_k| <= 702464 in plain mode), and one packed FADD of -1.5*2^23 leaves P -- one integer
// add on the ALU pipe per output instead of re-arming TMEM with a bias after every group (which needed a
// cluster-scope release per group and ran the C3-up GEMM at 2.2x the FP8 carrier's time, bench r2s).
// The MMA of group g+1 overlaps the promotion of group g (two TMEM buffers).  In plain mode (the
// per-channel A4W4 baseline of P:322) the MMA accumulates all K into one buffer per tile instead.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace rrs {

// Optional timeline (bench/micro/gemm_trace.cu builds this file with -DRRS_TRACE): %globaltimer at fixed
// points, per CTA, of the first tile's first 16 groups (rows 0..15), the first tile's last 8 groups
// (rows 16..23) and the second tile's first 8 groups (rows 24..31): [0] MMA after tempty wait, [1] after
// full wait, [2] after issue; [3]/[4] first promotion warp after tfull wait / after release; [5]/[6] last
// warp; [7] of rows 0/1 (tile 0) and 2/3 (tile 1): epilogue start / store issued.
#ifdef RRS_TRACE
__device__ unsigned long long g_gtrace[160][32][8];
__device__ __forceinline__ int gtrace_row(int it, int g, int G) {
  if (it == 0) return g < 16 ? g : (g >= G - 8 ? 16 + g - (G - 8) : -1);
  if (it == 1) return g < 8 ? 24 + g : -1;
  return -1;
}
__device__ __forceinline__ void gtrace(int row, int slot) {
  if (blockIdx.x < 160 && row >= 0 && row < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gtrace[blockIdx.x][row][slot] = t;
  }
}
#else
__device__ __forceinline__ int gtrace_row(int, int, int) { return -1; }
__device__ __forceinline__ void gtrace(int, int) {}
#endif

// Wait flavour of the per-group barriers (experiments: bench/micro/build.sh builds gemm_time with both)
#ifndef RRS_GEMM_SPIN_EPI
#define RRS_GEMM_SPIN_EPI 0
#endif
// 1: the 12 promotion warps of a CTA meet at a named barrier and ONE thread arrives on the leader's tempty
// (2 arrivals per buffer per pair instead of 24, 12 of them remote); 0: every warp arrives
#ifndef RRS_GEMM_ONE_RELEASE
#define RRS_GEMM_ONE_RELEASE 0
#endif
#ifndef RRS_GEMM_SPIN_MMA
#define RRS_GEMM_SPIN_MMA 0
#endif

namespace gemm {
constexpr int BM = 128;        // tokens per CTA    (TMEM lanes)
constexpr int BN = 240;        // outputs per tile  (TMEM columns per accumulator; 256-column slots)
constexpr int BK = 128;        // one smoothing group = one GEMM K-block
constexpr int NUM_EPI_WARPS = 12;
constexpr int EPI_COLS = BN / (NUM_EPI_WARPS / 4);  // columns per promotion thread (80)
constexpr int ACC_STRIDE = 256;  // TMEM column offset between the two accumulator buffers
constexpr int THREADS = 64 + NUM_EPI_WARPS * 32;
constexpr int MAX_G = 512;                 // smoothing groups per row: K / group <= 512

template <int kCta>
struct Cfg {
  static constexpr int B_ROWS = BN / kCta;                 // W rows loaded per CTA per group
  static constexpr int A_BYTES = BM * BK;                  // 16 KiB
  static constexpr int B_BYTES = B_ROWS * BK;              // 30 / 15 KiB (whole 8-row swizzle atoms)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = kCta == 1 ? 3 : 5;
  static constexpr int EPI_TILE_BYTES = 32 * EPI_COLS * 2;  // one promotion warp's bf16 Y sub-tile (TMA store)
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + NUM_EPI_WARPS * EPI_TILE_BYTES +
                                    1024 /*barriers*/ +
                                    MAX_G * 4 + 2 * BN * 4 + 2 * BM * 4 + 64 + 3 * BN * 4;
  static_assert(B_ROWS % 8 == 0 && (STAGES * A_BYTES) % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle atoms");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};
}  // namespace gemm

struct GemmParams {
  const float* x_scale;
  const float* s_group;
  const float* w_scale;
  int T, N, K, G;   // G = K / group smoothing groups
  int KB, gk;       // K-blocks of 128, MMA K-steps (of 32) per group
  int num_m, num_n, num_tiles;
  int num_mn;              // output tiles; num_tiles = num_mn * splits
  int splits, kps, gps;    // split-K (decode-sized T): K-blocks and groups per split
  int64_t split_stride;    // elements between the f32 partial outputs of consecutive splits
  float out_scale;
  void* Y;
  int64_t ldy;
  int32_t* P_debug;
  int y_tma;  // bf16 Y written by TMA tensor stores (16-byte aligned base, ldy % 8 == 0)
  int swiglu; // W rows interleaved (gate_i, up_i); Y[t][i] = bf16(silu(y_2i) * y_2i+1)
};

// kSub: the sub-channel A4W4 baseline of P:322 -- x_scale is alpha[G][T] and w_scale beta[G][N]
// (per token / per output row AND per group), Y = out_scale * sum_g alpha_gt * beta_gn * P_g; s_group unused.
template <bool kPlain, bool kF32Out, bool kDebug, int kCta, bool kFp8, bool kSub = false>
__global__ void __launch_bounds__(gemm::THREADS, 1)
rrs_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                const __grid_constant__ CUtensorMap tmap_y, GemmParams p) {
  using namespace gemm;
  using C = Cfg<kCta>;
  constexpr int STAGES = C::STAGES, A_BYTES = C::A_BYTES, B_BYTES = C::B_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B atoms) by offsetting the shared array itself, so the compiler keeps
  // the shared address space for every pointer derived from it (LDS/STS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* sY = smem + STAGES * STAGE_BYTES;  // [NUM_EPI_WARPS][32 rows][EPI_COLS] bf16 output staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sY + NUM_EPI_WARPS * C::EPI_TILE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* taddr_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* s_sm = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 1024);
  float* beta_sm = s_sm + MAX_G;     // [2][BN]   beta of the current tile (double-buffered by tile parity)
  float* xs_sm = beta_sm + 2 * BN;   // [2][BM]   alpha_t of the current / next tile's rows
  float* bsub_sm = xs_sm + 2 * BM + 16;  // [3][BN] sub-channel beta_g ring

  const uint32_t warp = ptx::warp_idx();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kCta == 2 ? ptx::cluster_ctarank() : 0u;  // position in the CTA pair
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_w);
    if constexpr (!kF32Out && !kDebug) ptx::prefetch_tmap(&tmap_y);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], kCta * (RRS_GEMM_ONE_RELEASE ? 1 : NUM_EPI_WARPS));  // only the leader's copy is used
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (kCta == 2) ptx::tmem_alloc2(taddr_slot, 512);
    else ptx::tmem_alloc(taddr_slot, 512);
  }
  if constexpr (kCta == 2) ptx::cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  ptx::pdl_wait();  // Xq8 / x_scale / s_group come from the prologue kernels (programmatic dependent launch)
  if (!kPlain && p.s_group) {
    for (int g = threadIdx.x; g < p.G; g += blockDim.x) s_sm[g] = p.s_group[g];
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *taddr_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x / kCta; tile < p.num_tiles; tile += gridDim.x / kCta) {
        const int mn = tile % p.num_mn, kb0 = (tile / p.num_mn) * p.kps;
        const int m_blk = mn % p.num_m, n_blk = mn / p.num_m;
        const int row0 = m_blk * BM * kCta + (int)rank * BM, wrow0 = n_blk * BN + (int)rank * C::B_ROWS;
        for (int kb = kb0; kb < kb0 + p.kps; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (kCta == 1) {
            ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            ptx::tma_load_2d(sA + stage * A_BYTES, &tmap_x, &full[stage], kb * BK, row0, ptx::kEvictNormal);
            ptx::tma_load_2d(sB + stage * B_BYTES, &tmap_w, &full[stage], kb * BK, wrow0, ptx::kEvictNormal);
          } else {
            // both CTAs' halves complete on the leader's barrier, which expects the pair's bytes
            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
            const uint32_t fb = ptx::mapa_shared(&full[stage], 0);
            ptx::tma_load_2d_pair(sA + stage * A_BYTES, &tmap_x, fb, kb * BK, row0, ptx::kEvictNormal);
            ptx::tma_load_2d_pair(sB + stage * B_BYTES, &tmap_w, fb, kb * BK, wrow0, ptx::kEvictNormal);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (pair leader)
    // one thread runs the whole loop: no warp-synchronous step between the barrier waits and the issue
    constexpr uint32_t idesc = kFp8 ? ptx::idesc_e4m3(BM * kCta, BN) : ptx::idesc_i8(BM * kCta, BN);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc_iter = 0;  // number of accumulator buffers filled so far
    int it = 0;             // local tile counter (timeline only)
    const uint64_t a_desc0 = ptx::smem_desc_sw128(sA), b_desc0 = ptx::smem_desc_sw128(sB);
    // smoothing groups of gk = group / 32 MMA K-steps: 4 for the paper's 128 = one K-block; the other
    // Table-4 sizes span several K-blocks (256+) or close inside one (32, 64)
    const int gk = p.gk;
    auto wait_tempty = [&](uint32_t b) {
      // a new accumulation into buffer b: use u = acc_iter >> 1 of it needs the u-th release (completion #u
      // of tempty[b]); the releases come from both CTAs of a pair (cluster-scope acquire for int8)
      if constexpr (RRS_GEMM_SPIN_MMA) ptx::mbar_wait_spin(&tempty[b], (acc_iter >> 1) & 1);
      else ptx::mbar_wait(&tempty[b], (acc_iter >> 1) & 1);
    };
    auto wait_full = [&]() {
      if constexpr (RRS_GEMM_SPIN_MMA) ptx::mbar_wait_spin(&full[stage], phase);
      else ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
    };
    auto mma = [&](uint32_t d, uint64_t a_desc, uint64_t b_desc, int k, uint32_t acc) {
      // advance 32 bytes (= 32 one-byte codes) along K inside the 128-byte swizzle row; a fresh sum per group
      if constexpr (kFp8) {
        if constexpr (kCta == 1) ptx::mma_f8(d, a_desc + 2 * k, b_desc + 2 * k, idesc, acc);
        else ptx::mma_f8_pair(d, a_desc + 2 * k, b_desc + 2 * k, idesc, acc);
      } else {
        if constexpr (kCta == 1) ptx::mma_i8(d, a_desc + 2 * k, b_desc + 2 * k, idesc, acc);
        else ptx::mma_i8_pair(d, a_desc + 2 * k, b_desc + 2 * k, idesc, acc);
      }
    };
    auto commit = [&](uint64_t* bar) {
      if constexpr (kCta == 1) ptx::mma_commit(bar);
      else ptx::mma_commit_pair(bar, 0x3);
    };
    if (kPlain || gk >= 4) {
      // whole K-blocks per group (the hot path): 4 MMAs back to back per K-block
      const int gpb = kPlain ? p.kps : gk / 4;  // K-blocks per accumulation
      for (int tile = blockIdx.x / kCta; leader && lane == 0 && tile < p.num_tiles; tile += gridDim.x / kCta) {
        int kin = 0;  // K-blocks into the current accumulation
        for (int kb = 0; kb < p.kps; ++kb, it += (kb == p.kps)) {
          const int trow = gtrace_row(it, kb, p.kps);
          const uint32_t b = acc_iter & 1;
          if (kin == 0) wait_tempty(b);
          gtrace(trow, 0);
          wait_full();
          gtrace(trow, 1);
          // descriptor start addresses advance in 16-byte units: stage offsets, then 32 bytes per K step
          const uint64_t a_desc = a_desc0 + (uint64_t)((stage * A_BYTES) >> 4);
          const uint64_t b_desc = b_desc0 + (uint64_t)((stage * B_BYTES) >> 4);
          const uint32_t d = tmem_base + b * ACC_STRIDE;
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) mma(d, a_desc, b_desc, k, (kin > 0 || k > 0) ? 1u : 0u);
          // the SMEM stage is free once these MMAs complete (a second commit per group costs ~18 ns of
          // tensor-pipe time, but freeing the stage from a promotion thread instead was slower)
          commit(&empty[stage]);
          if (++kin == gpb) {  // accumulation complete: hand the buffer to the promotion warps
            commit(&tfull[b]);
            ++acc_iter;
            kin = 0;
          }
          gtrace(trow, 2);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    } else {
      // groups of 32 or 64 codes: gk = 1 or 2 MMA K-steps, several groups per K-block
      int ks = 0;  // K-steps of the current group issued so far
      for (int tile = blockIdx.x / kCta; leader && lane == 0 && tile < p.num_tiles; tile += gridDim.x / kCta) {
        for (int kb = 0; kb < p.kps; ++kb) {
          wait_full();
          const uint64_t a_desc = a_desc0 + (uint64_t)((stage * A_BYTES) >> 4);
          const uint64_t b_desc = b_desc0 + (uint64_t)((stage * B_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            const uint32_t b = acc_iter & 1;
            if (ks == 0) {
              wait_tempty(b);
              ptx::tc_fence_after();
            }
            mma(tmem_base + b * ACC_STRIDE, a_desc, b_desc, k, ks > 0 ? 1u : 0u);
            if (++ks == gk) {
              commit(&tfull[b]);
              ++acc_iter;
              ks = 0;
            }
          }
          commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ promotion + epilogue
    constexpr uint32_t kBias = 0x4B400000u;  // bits of 1.5 * 2^23
    const int ew = warp - 2;                 // 0..15
    const int quad = warp & 3;               // TMEM lane quadrant this warp may access
    const int half = ew >> 2;                // column quarter of the 256-wide tile
    const int row_in_tile = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    ptx::tc_fence_before();
    __syncwarp();
    // buffer releases go to the pair leader's tempty barriers
    const uint32_t tempty_addr0 = kCta == 2 ? ptx::mapa_shared(&tempty[0], 0) : ptx::smem_u32(&tempty[0]);
    const uint32_t tempty_addr1 = kCta == 2 ? ptx::mapa_shared(&tempty[1], 0) : ptx::smem_u32(&tempty[1]);
    [[maybe_unused]] const int et0 = (int)threadIdx.x - 64;
    // release of an accumulator buffer to the pair leader's MMA thread (after this thread's tcgen05.ld/st)
    auto release = [&](uint32_t addr) {
      ptx::tc_fence_before();
#if RRS_GEMM_ONE_RELEASE
      asm volatile("bar.sync 3, %0;" ::"n"(NUM_EPI_WARPS * 32));
      if (et0 == 0) {
#else
      __syncwarp();
      if (lane == 0) {
#endif
        ptx::mbar_arrive_remote(addr);
      }
    };
    release(tempty_addr0);
    release(tempty_addr1);
    const float2 neg_bias2 = make_float2(-12582912.0f, -12582912.0f);  // -1.5*2^23
    uint32_t acc_iter = 0;
    int it = 0;  // local tile counter
    const int tile_stride = gridDim.x / kCta;
    const int et = (int)threadIdx.x - 64;  // 0 .. 383: epilogue thread index
    // alpha_t (per row) and beta_n (per column) reach shared memory through cp.async, never through
    // registers: alpha one tile ahead (it is folded into every group's scale), beta during the tile's K loop.
    // Completion: cp.async.wait_group 0 + the epilogue's named barrier.
    auto fetch_xs = [&](int tile, int buf) {
      if (et < BM) {
        const int r = ((tile % p.num_mn) % p.num_m) * BM * kCta + (int)rank * BM + et;
        const bool ok = !kSub && tile < p.num_tiles && p.x_scale && r < p.T;
        ptx::cp_async4(xs_sm + buf * BM + et, ok ? p.x_scale + r : p.x_scale, ok ? 4u : 0u);
      }
    };
    fetch_xs(blockIdx.x / kCta, 0);
    ptx::cp_async_commit();
    ptx::cp_async_wait_all();
    asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32));
    for (int tile = blockIdx.x / kCta; tile < p.num_tiles; tile += tile_stride, ++it) {
      const int mn = tile % p.num_mn, split = tile / p.num_mn;
      const int m_blk = mn % p.num_m, n_blk = mn / p.num_m;
      const int row = m_blk * BM * kCta + (int)rank * BM + row_in_tile;
      const int col0 = n_blk * BN + half * EPI_COLS;
      // rs = alpha_t * out_scale is folded into every group's scale (acc = sum_g fl(s_g * rs) * P_g), so the
      // epilogue is a single multiply by beta_n
      const float rs = kSub ? p.out_scale : xs_sm[(it & 1) * BM + row_in_tile] * p.out_scale;
      if (et < BN) {
        const int n = n_blk * BN + et;
        if constexpr (kSub) {
          beta_sm[(it & 1) * BN + et] = 1.0f;  // beta_gn already applied per group
        } else {
          const bool ok = p.w_scale && n < p.N;
          ptx::cp_async4(beta_sm + (it & 1) * BN + et, ok ? p.w_scale + n : p.w_scale, ok ? 4u : 0u);
        }
      }
      fetch_xs(tile + tile_stride, (it + 1) & 1);
      ptx::cp_async_commit();

      float2 acc2[EPI_COLS / 2];  // acc pairs (columns 2i, 2i+1 of this thread's EPI_COLS)
#pragma unroll
      for (int c = 0; c < EPI_COLS / 2; ++c) acc2[c] = make_float2(0.0f, 0.0f);
      if (it < 2 && lane == 0 && ew == 0) gtrace(8 * it + 6, 7);
      const int ngroups = kPlain ? 1 : p.gps;
      const float* s_split = s_sm + split * p.gps;  // this split's groups
      // sub-channel: beta_g of this tile's columns staged in a 3-slot shared ring by cp.async two groups
      // ahead (one named barrier per group), alpha_g of this thread's row prefetched one group ahead
      auto fetch_bsub = [&](int g) {
        if (g < ngroups && et < BN) {
          const int n = n_blk * BN + et;
          const bool ok = n < p.N;
          const float* src = p.w_scale + (int64_t)(split * p.gps + g) * p.N + (ok ? n : 0);
          ptx::cp_async4(bsub_sm + (g % 3) * BN + et, src, ok ? 4u : 0u);
        }
        ptx::cp_async_commit();  // possibly empty: one commit group per call keeps the wait counts uniform
      };
      auto load_alpha = [&](int g) {
        return (g < ngroups && row < p.T) ? __ldg(p.x_scale + (int64_t)(split * p.gps + g) * p.T + row) : 0.0f;
      };
      float alpha_next = 0.0f;
      if constexpr (kSub) {
        fetch_bsub(0);
        fetch_bsub(1);
        alpha_next = load_alpha(0);
      }
      for (int g = 0; g < ngroups; ++g) {
        const uint32_t b = acc_iter & 1;
        // RRS: a buffer lands every group, spin for the lowest wake-up latency; plain: once per tile, sleep
        if constexpr (kPlain || !RRS_GEMM_SPIN_EPI) ptx::mbar_wait(&tfull[b], (acc_iter >> 1) & 1);
        else ptx::mbar_wait_spin(&tfull[b], (acc_iter >> 1) & 1);
        ptx::tc_fence_after();
        // group acc_iter's MMAs are complete, so its SMEM stage (acc_iter % STAGES in the producer's order)
        // is free: one thread per CTA releases it to this CTA's producer
        const bool trace_me = lane == 0 && (ew == 0 || ew == NUM_EPI_WARPS - 1);
        const int trow = gtrace_row(it, g, p.G);
        if (trace_me) gtrace(trow, ew == 0 ? 3 : 5);
        const float s = kPlain ? rs : s_split[g] * rs;
        const float2 s2 = make_float2(s, s);
        const uint32_t tbase = tmem_base + lane_off + b * ACC_STRIDE + half * EPI_COLS;
#if defined(RRS_TRACE) && defined(RRS_GEXP) && RRS_GEXP == 1
        if constexpr (kFp8 && !kDebug) {  // timeline experiment: no TMEM readout at all
          release(b ? tempty_addr1 : tempty_addr0);
          acc2[g % (EPI_COLS / 2)].x += s;
        } else
#endif
        if constexpr (kSub) {
          // sub-channel: every element has its own scale alpha_gt * beta_gn (beta read through L1, the 32 lanes
          // of a warp share its 80 columns), applied per group before the FP32 accumulation
          const float a = alpha_next * rs;
          alpha_next = load_alpha(g + 1);
          ptx::cp_async_wait_1();  // this thread's copies of group g have landed (g + 1 may be in flight)
          asm volatile("bar.sync 2, %0;" ::"n"(NUM_EPI_WARPS * 32));  // ... and every thread's
          const float4* bg4 = reinterpret_cast<const float4*>(bsub_sm + (g % 3) * BN + half * EPI_COLS);
          fetch_bsub(g + 2);  // into the slot read in iteration g - 1, which every warp has left
#pragma unroll
          for (int cc = 0; cc < EPI_COLS / 16; ++cc) {
            uint32_t r[16];
            RRS_TMEM_LD16(tbase + cc * 16, r);
            RRS_TMEM_WAIT_LD16(r);
            if (cc == EPI_COLS / 16 - 1) {  // every column of this buffer is in registers: release it
              release(b ? tempty_addr1 : tempty_addr0);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 bv = bg4[cc * 4 + q];
              const float2 s01 = __fmul2_rn(make_float2(a, a), make_float2(bv.x, bv.y));
              const float2 s23 = __fmul2_rn(make_float2(a, a), make_float2(bv.z, bv.w));
              acc2[cc * 8 + 2 * q] = __ffma2_rn(s01, make_float2(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1])),
                                                acc2[cc * 8 + 2 * q]);
              acc2[cc * 8 + 2 * q + 1] = __ffma2_rn(
                  s23, make_float2(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])), acc2[cc * 8 + 2 * q + 1]);
            }
          }
        } else if constexpr (!kDebug) {
          // software-pipelined: chunk c+1 is in flight while chunk c is accumulated; the buffer is released
          // as soon as the last chunk has landed in registers
          constexpr int NCH = EPI_COLS / 16;
          uint32_t ra[16], rb[16];
          RRS_TMEM_LD16(tbase, ra);
          RRS_TMEM_WAIT_LD16(ra);
#pragma unroll
          for (int cc = 0; cc < NCH; ++cc) {
            uint32_t(&cur)[16] = (cc & 1) ? rb : ra;
            uint32_t(&nxt)[16] = (cc & 1) ? ra : rb;
            if (cc + 1 < NCH) RRS_TMEM_LD16(tbase + (cc + 1) * 16, nxt);
#if defined(RRS_TRACE) && defined(RRS_GEXP) && RRS_GEXP == 2
            for (int j = 0; j < 8; ++j) acc2[cc * 8 + j].x = __uint_as_float(__float_as_uint(acc2[cc * 8 + j].x) ^ cur[2 * j] ^ cur[2 * j + 1]);
            if (false)
#endif
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // acc += s_g * P_g (R14); the FP8 carrier's P_g is an exact float
              float2 f = make_float2(__uint_as_float(cur[2 * j]), __uint_as_float(cur[2 * j + 1]));
              if constexpr (!kFp8)  // int8: bits(P + 0x4B400000) - 1.5*2^23 = P exactly (|P| < 2^22)
                f = __fadd2_rn(make_float2(__uint_as_float(cur[2 * j] + kBias), __uint_as_float(cur[2 * j + 1] + kBias)),
                               neg_bias2);
              acc2[cc * 8 + j] = __ffma2_rn(s2, f, acc2[cc * 8 + j]);
            }
            if (cc + 1 < NCH) {
              RRS_TMEM_WAIT_LD16(nxt);
              if (cc + 2 == NCH) {  // all chunks of this buffer are in registers: release it
                release(b ? tempty_addr1 : tempty_addr0);
                if (trace_me) gtrace(trow, ew == 0 ? 4 : 6);
              }
            }
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < EPI_COLS / 16; ++cc) {
            uint32_t r[16];
            RRS_TMEM_LD16(tbase + cc * 16, r);
            RRS_TMEM_WAIT_LD16(r);
            if (cc == EPI_COLS / 16 - 1) {
              // every column of this buffer is in registers: release it before the last chunk's math
              release(b ? tempty_addr1 : tempty_addr0);
            }
            if (kDebug && row < p.T) {
              const int gg = kPlain ? 0 : g;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int n = col0 + cc * 16 + j;
                const int32_t P = kFp8 ? __float2int_rn(__uint_as_float(r[j])) : (int32_t)r[j];
                if (n < p.N) p.P_debug[((int64_t)gg * p.T + row) * p.N + n] = P;
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float2 f = make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
              // int8 carrier: bits(P + 0x4B400000) = 1.5*2^23 + P, minus 1.5*2^23 = P exactly for |P| < 2^22; FP8
              // carrier: P is already an exact float.  Then acc += s_g * P (R14).
              if constexpr (!kFp8)
                f = __fadd2_rn(make_float2(__uint_as_float(r[2 * j] + kBias), __uint_as_float(r[2 * j + 1] + kBias)),
                               neg_bias2);
              acc2[cc * 8 + j] = __ffma2_rn(s2, f, acc2[cc * 8 + j]);
            }
          }
        }
        ++acc_iter;
      }
      // ---- epilogue: Y = acc * beta_n  (acc already carries alpha_t * out_scale)
      const bool trace_epi = it < 2 && lane == 0 && ew == 0;
      if (trace_epi) gtrace(8 * it, 7);
      // this tile's beta and the next tile's alpha have landed (every thread's copies: wait + named barrier);
      // the buffers written next were last read before this barrier
      ptx::cp_async_wait_all();
      asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32));
      if (trace_epi) gtrace(8 * it + 1, 7);
      const float2* beta2 = reinterpret_cast<const float2*>(beta_sm + (it & 1) * BN + half * EPI_COLS);
      if (p.Y != nullptr && (row < p.T || (!kF32Out && !kDebug && p.y_tma))) {
        if constexpr (kF32Out || kDebug) {
          float* yrow = reinterpret_cast<float*>(p.Y) + split * p.split_stride + (int64_t)row * p.ldy;
#pragma unroll
          for (int c = 0; c < EPI_COLS; c += 4) {
            const int n = col0 + c;
            const float2 lo = __fmul2_rn(acc2[c / 2], beta2[c / 2]), hi = __fmul2_rn(acc2[c / 2 + 1], beta2[c / 2 + 1]);
            if (n + 3 < p.N) {
              *reinterpret_cast<float4*>(yrow + n) = make_float4(lo.x, lo.y, hi.x, hi.y);
            } else {
              if (n < p.N) yrow[n] = lo.x;
              if (n + 1 < p.N) yrow[n + 1] = lo.y;
              if (n + 2 < p.N) yrow[n + 2] = hi.x;
            }
          }
        } else {
          // bf16: with TMA, this warp's 32 x 80 sub-tile goes through shared memory and one tensor store
          // (coalesced, asynchronous, clipped at the T / N edges by the tensor map); else 16-byte row stores
          auto pack8 = [&](int c, uint32_t (&w)[4]) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 v = __fmul2_rn(acc2[c / 2 + h], beta2[c / 2 + h]);
              const __nv_bfloat162 bb = __floats2bfloat162_rn(v.x, v.y);
              w[h] = *reinterpret_cast<const uint32_t*>(&bb);
            }
          };
          if (p.y_tma) {
            uint8_t* my = sY + ew * C::EPI_TILE_BYTES;
            if (lane == 0) ptx::bulk_wait_group_read0();  // the previous tile's store has read this buffer
            __syncwarp();
            if (trace_epi) gtrace(8 * it + 2, 7);
#pragma unroll
            for (int c = 0; c < EPI_COLS; c += 8) {
              uint32_t w[4];
              pack8(c, w);
              *reinterpret_cast<uint4*>(my + lane * (EPI_COLS * 2) + c * 2) = make_uint4(w[0], w[1], w[2], w[3]);
            }
            ptx::fence_proxy_async_shared();
            if (trace_epi) gtrace(8 * it + 3, 7);
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&tmap_y, my, col0, m_blk * BM * kCta + (int)rank * BM + quad * 32);
              ptx::bulk_commit_group();
              if (trace_epi) gtrace(8 * it + 4, 7);
            }
          } else if (p.swiglu) {
            // fused SwiGLU: this thread's column pairs (2i, 2i+1) are (gate_i, up_i), so
            // h_i = silu(g) * u = g / (1 + e^-g) * u in f32, rounded once to bf16; 8 outputs per 16-byte store
            __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.Y) + (int64_t)row * p.ldy;
            auto swiglu1 = [](float2 v) { return v.x / (1.0f + expf(-v.x)) * v.y; };
#pragma unroll
            for (int c = 0; c < EPI_COLS; c += 16) {
              uint32_t w[4];
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float h0 = swiglu1(__fmul2_rn(acc2[c / 2 + 2 * h], beta2[c / 2 + 2 * h]));
                const float h1 = swiglu1(__fmul2_rn(acc2[c / 2 + 2 * h + 1], beta2[c / 2 + 2 * h + 1]));
                const __nv_bfloat162 bb = __floats2bfloat162_rn(h0, h1);
                w[h] = *reinterpret_cast<const uint32_t*>(&bb);
              }
              const int i = (col0 + c) >> 1, nh = p.N >> 1;
              if (i + 7 < nh) {
                *reinterpret_cast<uint4*>(hrow + i) = make_uint4(w[0], w[1], w[2], w[3]);
              } else {
                const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(w);
                for (int h = 0; h < 8; ++h)
                  if (i + h < nh) hrow[i + h] = e[h];
              }
            }
          } else {
            __nv_bfloat16* yrow = reinterpret_cast<__nv_bfloat16*>(p.Y) + (int64_t)row * p.ldy;
#pragma unroll
            for (int c = 0; c < EPI_COLS; c += 8) {
              uint32_t w[4];
              pack8(c, w);
              const int n = col0 + c;
              if (n + 7 < p.N) {
                *reinterpret_cast<uint4*>(yrow + n) = make_uint4(w[0], w[1], w[2], w[3]);
              } else {
                const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(w);
                for (int h = 0; h < 8; ++h)
                  if (n + h < p.N) yrow[n + h] = e[h];
              }
            }
          }
        }
      }
      if (trace_epi) gtrace(8 * it + 5, 7);
    }
  }
  if constexpr (!kF32Out && !kDebug) {
    if (p.y_tma && warp >= 2 && lane == 0) ptx::bulk_wait_group0();  // Y stores complete before the CTA retires
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kCta == 2) ptx::cluster_sync();  // the peer's MMAs / arrives are done before TMEM goes away
  if (warp == 1) {
    if constexpr (kCta == 2) ptx::tmem_dealloc2(tmem_base, 512);
    else ptx::tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2-D int8 K-major operand [rows][K] with a (box_rows x 128-byte) box and 128-byte swizzle
static bool make_tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D bf16 row-major Y [T][ldy] (N valid columns), written in (32 rows x EPI_COLS) boxes; the map clips the
// T / N edges so ragged tiles need no masking
static bool make_tmap_y(CUtensorMap* m, void* base, int64_t T, int64_t N, int64_t ldy) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)T};
  cuuint64_t strides[1] = {(cuuint64_t)(ldy * 2)};
  cuuint32_t box[2] = {(cuuint32_t)gemm::EPI_COLS, 32u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool kPlain, bool kF32, bool kDebug, int kCta, bool kFp8, bool kSub = false>
static cudaError_t launch_variant(const CUtensorMap& tx, const CUtensorMap& tw, const CUtensorMap& ty,
                                  const GemmParams& p, int grid,
                                  cudaStream_t st) {
  auto kern = rrs_gemm_kernel<kPlain, kF32, kDebug, kCta, kFp8, kSub>;
  constexpr int smem = gemm::Cfg<kCta>::SMEM_BYTES;
  cudaError_t e = prepare_kernel(kern, smem, gemm::THREADS);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap our setup with the prologue's tail
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;  // CTA pairs for cta_group::2
  attr[1].val.clusterDim.x = kCta;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, tx, tw, ty, p);
}

template <int kCta, bool kFp8>
static cudaError_t launch_cta(const GemmArgs& a, int nsm, cudaStream_t st) {
  using namespace gemm;
  CUtensorMap tx, tw;
  if (!make_tmap(&tx, a.Xq8, a.T, a.K, BM) || !make_tmap(&tw, a.Wq8, a.N, a.K, Cfg<kCta>::B_ROWS))
    return cudaErrorInvalidValue;
  GemmParams p;
  p.x_scale = a.x_scale;
  p.s_group = a.s_group;
  p.w_scale = a.w_scale;
  p.T = (int)a.T;
  p.N = (int)a.N;
  p.K = (int)a.K;
  p.G = (int)(a.K / a.group);
  p.KB = (int)(a.K / BK);
  p.gk = a.group / 32;
  p.num_m = (int)((a.T + BM * kCta - 1) / (BM * kCta));
  p.num_n = (int)((a.N + BN - 1) / BN);
  p.num_mn = p.num_m * p.num_n;
  p.splits = a.splits;
  p.kps = p.KB / a.splits;
  p.gps = p.G / a.splits;
  p.split_stride = (int64_t)a.T * a.ldy;
  p.num_tiles = p.num_mn * a.splits;
  // a split owns whole K-blocks and whole groups; split partials are f32 (reduced by reduce_splits_kernel)
  if (a.splits < 1 || p.KB % a.splits || p.G % a.splits || (a.splits > 1 && (a.plain || a.y_dtype != 1 || a.swiglu)))
    return cudaErrorInvalidValue;
  p.out_scale = a.out_scale;
  p.Y = a.Y;
  p.ldy = a.ldy;
  p.P_debug = a.P_debug;
  // bf16 output tile stores through TMA when the layout allows it (else per-thread 16-byte stores)
  CUtensorMap ty;
  memset(&ty, 0, sizeof(ty));
  p.y_tma = 0;
  p.swiglu = a.swiglu ? 1 : 0;
  if (a.swiglu && (a.y_dtype == 1 || a.plain || a.P_debug || a.N % 2)) return cudaErrorInvalidValue;
#ifndef RRS_GEMM_Y_TMA
#define RRS_GEMM_Y_TMA 1  // experiment knob (bench/micro): 0 = per-thread 16-byte row stores for bf16 Y
#endif
  // (a TMA store writes whole 16-byte chunks at the right edge of the tensor, so it is only used when the output
  // width is a multiple of 8 bf16: columns past N belong to the caller, e.g. a column slice of a wider matrix.
  // The fused SwiGLU output uses per-thread 16-byte stores: its 40-column TMA boxes lost every other box.)
  if (RRS_GEMM_Y_TMA && !a.swiglu && a.Y && a.y_dtype != 1 && !a.P_debug && a.ldy % 8 == 0 && a.N % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(a.Y) & 15) == 0)
    p.y_tma = make_tmap_y(&ty, a.Y, a.T, a.N, a.ldy) ? 1 : 0;
  const int grid = std::min(p.num_tiles, nsm / kCta) * kCta;
  const bool f32 = a.y_dtype == 1;
  if (a.P_debug) return launch_variant<false, true, true, kCta, kFp8>(tx, tw, ty, p, grid, st);
  if (a.subchannel) {
    if constexpr (kFp8)
      return f32 ? launch_variant<false, true, false, kCta, true, true>(tx, tw, ty, p, grid, st)
                 : launch_variant<false, false, false, kCta, true, true>(tx, tw, ty, p, grid, st);
    return cudaErrorInvalidValue;  // the baseline is built for the FP8 carrier only
  }
  if (a.plain)
    return f32 ? launch_variant<true, true, false, kCta, kFp8>(tx, tw, ty, p, grid, st)
               : launch_variant<true, false, false, kCta, kFp8>(tx, tw, ty, p, grid, st);
  return f32 ? launch_variant<false, true, false, kCta, kFp8>(tx, tw, ty, p, grid, st)
             : launch_variant<false, false, false, kCta, kFp8>(tx, tw, ty, p, grid, st);
}

cudaError_t launch_gemm(const GemmArgs& a, int nsm, cudaStream_t st) {
  using namespace gemm;
  if (a.T <= 0) return cudaSuccess;
  if (a.group < 32 || a.group % 32 || a.K % a.group || a.K / a.group > MAX_G || a.K % BK) return cudaErrorInvalidValue;
  // CTA pairs (M = 256) once there are enough tokens to fill them; single CTAs for decode-sized T
  if (a.fp8) return a.T > BM ? launch_cta<2, true>(a, nsm, st) : launch_cta<1, true>(a, nsm, st);
  return a.T > BM ? launch_cta<2, false>(a, nsm, st) : launch_cta<1, false>(a, nsm, st);
}

// Split-K (decode-sized T): Y[t][n] = sum over splits s = 0, 1, ... (fixed order, deterministic, R15) of the
// f32 partials part[s][t][n] (each already acc * beta); f32 or bf16 (RNE) out.  4 columns per thread.
__global__ void reduce_splits_kernel(const float* __restrict__ part, int splits, int64_t T, int64_t N,
                                     void* __restrict__ Y, int y_bf16, int64_t ldy) {
  const int64_t nq = N / 4, total = T * nq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / nq, n = (i % nq) * 4;
    float4 acc = reinterpret_cast<const float4*>(part + t * N + n)[0];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(part + (s * T + t) * N + n)[0];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (y_bf16) {
      const __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 w;
      w.x = *reinterpret_cast<const uint32_t*>(&lo);
      w.y = *reinterpret_cast<const uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(Y) + t * ldy + n) = w;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(Y) + t * ldy + n) = acc;
    }
  }
}

cudaError_t launch_reduce_splits(const float* part, int splits, int64_t T, int64_t N, void* Y, int y_dtype,
                                 int64_t ldy, cudaStream_t st) {
  if (N % 4) return cudaErrorInvalidValue;
  const int64_t total = T * (N / 4);
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 8);
  reduce_splits_kernel<<<blocks, threads, 0, st>>>(part, splits, T, N, Y, y_dtype == 1 ? 0 : 1, ldy);
  return cudaGetLastError();
}

// Y[t][r*ns + j] = gather[r][t][j]  (all-gathered column shards -> row-major Y), 16-byte chunks
__global__ void relayout_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t T,
                                int64_t shard_bytes, int world, int64_t ldy_bytes) {
  const int64_t chunks_per_row = shard_bytes / 16;
  const int64_t total = (int64_t)world * T * chunks_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % chunks_per_row;
    const int64_t t = (i / chunks_per_row) % T;
    const int64_t r = i / (chunks_per_row * T);
    const uint4 v = reinterpret_cast<const uint4*>(src + (r * T + t) * shard_bytes)[c];
    reinterpret_cast<uint4*>(dst + t * ldy_bytes + r * shard_bytes)[c] = v;
  }
}

cudaError_t launch_relayout_shards(const void* src, void* dst, int64_t T, int64_t n_shard, int world, int64_t ldy,
                                   int elem_bytes, cudaStream_t st) {
  const int64_t shard_bytes = n_shard * elem_bytes;
  if (shard_bytes % 16 || (ldy * elem_bytes) % 16) return cudaErrorInvalidValue;
  const int64_t total = world * T * (shard_bytes / 16);
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 8);
  if (blocks == 0) return cudaSuccess;
  relayout_kernel<<<blocks, threads, 0, st>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), T,
                                              shard_bytes, world, ldy * elem_bytes);
  return cudaGetLastError();
}

}  // namespace rrs

// RRS runtime prologue (rows a1-a6 of SURVEY.md §8) and offline weight preparation (a7), sm_100a.
//
//   fwht_colmax_kernel  : X~ = X.H (exact, fwht.cuh), written once as f32 [T][K] (L2-resident at the
//                         prefill shapes), and c_j = max_t |X~_tj| over all T tokens (Eq. 1) via
//                         per-thread running maxima + one atomicMax per column per CTA on the float bits
//                         (valid because |x| >= +0).  Rows arrive by TMA bulk copies, double-buffered, so
//                         the next tile's HBM read overlaps this tile's FP64 butterflies.
//   smooth_quant_kernel : s_g = max_{j' in g} c[perm[j']] (0 -> 1, R8), Z = X~[perm] * fl(1/s_g)
//                         (Eq. 2, R9), per-token RTN INT4 (R9-R11), pack (D4) and the int8 GEMM
//                         operand.  With chan_max == nullptr it is the weight path (a7): no smoothing
//                         (W is permuted, never scaled).
//   perm_rank_kernel    : offline reorder helper (R5): perm = argsort(c) descending, ties ascending.
#include <algorithm>
#include <cstdlib>
#include <atomic>

#include "fwht.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace rrs {

// Optional per-CTA timeline (bench/micro/prologue_trace.cu builds this file with -DRRS_TRACE): thread 0
// records %globaltimer at fixed points into g_trace[kernel][cta][slot].
#ifdef RRS_TRACE
__device__ unsigned long long g_trace[3][1024][16];
__device__ unsigned long long g_trace_clk[3][1024][16];  // the SM's clock64 at the same points (effective SM clock)
RRS_DEVICE void trace(int k, int slot) {
  if (threadIdx.x == 0 && blockIdx.x < 1024 && slot < 16) {
    unsigned long long t, c;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory");
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) :: "memory");
    g_trace[k][blockIdx.x][slot] = t;
    g_trace_clk[k][blockIdx.x][slot] = c;
  }
}
void copy_prologue_trace(void* dst, size_t bytes) { cudaMemcpyFromSymbol(dst, g_trace, bytes); }
void copy_prologue_trace_clk(void* dst, size_t bytes) { cudaMemcpyFromSymbol(dst, g_trace_clk, bytes); }
#else
RRS_DEVICE void trace(int, int) {}
#endif

// ------------------------------------------------------------------------------ a1 + a2

template <int K>
struct ColmaxSmem {
  using P = FwhtPlan<K>;
  static constexpr int TILE_D = ((P::TILE_PAD * 8 + 127) / 128) * 128;  // padded fp64 transpose tile
  static constexpr int STAGE = P::TILE * 2;     // one bf16 tile
  static constexpr int BYTES = TILE_D + 2 * STAGE + 64 + 64 * 4;  // + 5 barriers (40 B), reduction scratch
  static_assert(2 * P::TILE * 4 <= TILE_D && K * 4 <= 2 * STAGE, "fused quantisation staging");
};

// CTAs that combine their column maxima through DSMEM before the atomics.  2^m plans run several CTAs per SM,
// so clusters of 8 pack densely; the 28*2^m plan runs one 256-thread CTA per SM, where a cluster of 8 must fit
// inside one GPC and only 15 such clusters (120 of 148 SMs) are co-resident -- pairs use every SM.
template <int K>
__host__ __device__ constexpr int colmax_cluster() { return FwhtPlan<K>::kPow2 ? 8 : 2; }

// The FWHT pass (rows a1-a2): every CTA of the (persistent, clustered) grid transforms its rows, writes X~
// f32 and, unless chan_max_bits is null, folds its column maxima into chan_max (DSMEM cluster reduction +
// one atomicMax per column per cluster).  Ends with a cluster barrier.  Every thread must call it.
template <int K, bool kFinalClusterSync = true>
RRS_DEVICE void fwht_phase(const uint16_t* __restrict__ X, int64_t T, unsigned* __restrict__ chan_max_bits,
                           float* __restrict__ Xr, uint8_t* smem) {
  using P = FwhtPlan<K>;
  using S = ColmaxSmem<K>;
  double* sm = reinterpret_cast<double*>(smem);
  uint16_t* stage = reinterpret_cast<uint16_t*>(smem + S::TILE_D);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::TILE_D + 2 * S::STAGE);
  const int64_t ntiles = (T + P::R - 1) / P::R;
  trace(0, 0);

  auto issue = [&](int64_t tile, int buf) {
    const int64_t rows = (T - tile * P::R) < P::R ? (T - tile * P::R) : P::R;
    const uint32_t bytes = (uint32_t)(rows * K * 2);
    ptx::mbar_arrive_expect_tx(&bar[buf], bytes);
    ptx::bulk_load(stage + buf * P::TILE, X + tile * P::R * K, bytes, &bar[buf]);
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < 5; ++b) ptx::mbar_init(&bar[b], 1);  // [0,1] this pass; [2..4] the fused quant pass
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  float cm[P::SLOTS];
#pragma unroll
  for (int j = 0; j < P::SLOTS; ++j) cm[j] = 0.0f;
  const bool act = out_active<P>(threadIdx.x);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    ptx::mbar_wait(&bar[buf], (it >> 1) & 1);
    trace(0, 1 + 2 * (it < 5 ? it : 5));
    double v[P::E];
    int rr = 0, tp = 0;
    // X~ stores and column maxima as the values are produced; the row and its pointer are fixed before the
    // transform, so every store is one base register plus a compile-time offset and nothing branches per element
    int rr0, tp0;
    tile_coords<P>((int)threadIdx.x, rr0, tp0);
    const int64_t row = tile * P::R + rr0;
    const bool live = act && row < T;
    float* xr = Xr + (live ? row : 0) * (int64_t)K + out_col<P>(tp0, 0);  // + a compile-time offset per register
    auto emit = [&](int j, float f) {
      cm[j] = live ? fmaxf(cm[j], fabsf(f)) : cm[j];
      if (live) xr[out_col<P>(0, j)] = f;
    };
    fwht_tile<P>(stage + buf * P::TILE, sm, v, rr, tp, emit);  // ends with __syncthreads: stage[buf] is free
    trace(0, 2 + 2 * (it < 5 ? it : 5));
    if (threadIdx.x == 0 && tile + 2 * (int64_t)gridDim.x < ntiles) issue(tile + 2 * (int64_t)gridDim.x, buf);
  }
  trace(0, 12);
  ptx::pdl_launch_dependents();
  if (chan_max_bits == nullptr) return;  // weight path: no column maxima (uniform over the cluster)
  // Column maxima: CTA -> shared memory, then the 8 CTAs of the cluster combine through DSMEM so each
  // column sees one global atomicMax per cluster instead of one per CTA.
  uint32_t* cmx = reinterpret_cast<uint32_t*>(smem);  // [K], reuses the transpose tile
  __syncthreads();
  for (int c = threadIdx.x; c < K; c += P::THREADS) cmx[c] = 0u;
  __syncthreads();
  if (act) {
    const int tp = P::kPow2 ? (int)threadIdx.x % P::TP2 : (int)threadIdx.x;  // columns do not depend on the row
#pragma unroll
    for (int j = 0; j < P::SLOTS; ++j) {
      if constexpr (P::R == 1) {
        cmx[out_col<P>(tp, j)] = __float_as_uint(cm[j]);  // each column is owned by exactly one thread
      } else {
        atomicMax(cmx + out_col<P>(tp, j), __float_as_uint(cm[j]));
      }
    }
  }
  ptx::cluster_sync();
  trace(0, 13);
  const uint32_t rank = ptx::cluster_ctarank();
  constexpr int SLICE = K / colmax_cluster<K>();
  constexpr int PER_THREAD = (SLICE + P::THREADS - 1) / P::THREADS;
  uint32_t mx[PER_THREAD];
#pragma unroll
  for (int i = 0; i < PER_THREAD; ++i) {  // all 8 x PER_THREAD remote loads in flight at once
    const int c = (int)rank * SLICE + threadIdx.x + i * P::THREADS;
    uint32_t m = 0u;
    if (threadIdx.x + i * P::THREADS < SLICE) {
#pragma unroll
      for (uint32_t r = 0; r < colmax_cluster<K>(); ++r) m = max(m, ptx::ld_dsmem_u32(cmx + c, r));
    }
    mx[i] = m;
  }
#pragma unroll
  for (int i = 0; i < PER_THREAD; ++i) {
    const int c = (int)rank * SLICE + threadIdx.x + i * P::THREADS;
    if (threadIdx.x + i * P::THREADS < SLICE) atomicMax(chan_max_bits + c, mx[i]);  // float bits of values >= +0
  }
  trace(0, 14);
  // keep this CTA's shared memory alive until every peer has read it (the fused kernel's grid barrier,
  // which starts with a cluster barrier, provides the same guarantee)
  if constexpr (kFinalClusterSync) ptx::cluster_sync();
  trace(0, 15);
}

template <int K>
__global__ void __cluster_dims__(colmax_cluster<K>(), 1, 1) __launch_bounds__(FwhtPlan<K>::THREADS, FwhtPlan<K>::MIN_BLOCKS)
fwht_colmax_kernel(const uint16_t* __restrict__ X, int64_t T, unsigned* __restrict__ chan_max_bits,
                   float* __restrict__ Xr) {
  extern __shared__ __align__(128) uint8_t smem[];
  fwht_phase<K>(X, T, chan_max_bits, Xr, smem);
}

// ------------------------------------------------------------------------------ a3 - a6 (and a7)

// max over the `width` consecutive lanes sharing a segment (width = power of two <= 32)
RRS_DEVICE float seg_max(float m, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

// GEMM operand byte of an INT4 code q in [-8, 7]: the code itself (int8 carrier) or its E4M3 encoding
// (FP8 carrier; every integer of magnitude <= 8 is exact in E4M3: 1.mmm x 2^e, e = floor(log2|q|)).
RRS_DEVICE uint32_t operand_byte(int q, bool e4m3) {
  if (!e4m3) return (uint32_t)(q & 0xFF);
  const uint32_t a = (uint32_t)(q < 0 ? -q : q);
  const uint32_t e = 31u - __clz(a | 1u);            // floor(log2 a) for a >= 1
  const uint32_t m = ((a << 3) >> e) & 7u;           // 3 fraction bits
  const uint32_t mag = a ? (((e + 7u) << 3) | m) : 0u;  // exponent bias 7
  return mag | (q < 0 ? 0x80u : 0u);
}


// ------------------------------------------------------------------------------ a3 - a6 building blocks

// This thread's 32 reordered positions j0..j0+31 -> perm entries (an offline input).
RRS_DEVICE void load_perm32(const int32_t* __restrict__ perm, int j0, int (&pj)[32]) {
  const int4* pp = reinterpret_cast<const int4*>(perm + j0);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int4 w = __ldg(pp + q);
    pj[4 * q] = w.x; pj[4 * q + 1] = w.y; pj[4 * q + 2] = w.z; pj[4 * q + 3] = w.w;
  }
}

// s_g = max_{j' in g} c[perm[j']] (the group/32 consecutive threads of a group -- 4 for the paper's 128,
// P:189) from chan_max staged in shared memory; 0 -> 1 (R8); returns fl(1/s_g) (R9).  CTA 0's first tile row
// publishes s_group.  group in {32, 64, ..., 1024}, a divisor of the row's thread count x 32.
RRS_DEVICE float group_inv_scale(const float* cms, const int (&pj)[32], int j0, bool publish, float* s_group_out,
                                 int group) {
  float m = 0.0f;
#pragma unroll
  for (int k = 0; k < 32; ++k) m = fmaxf(m, cms[pj[k]]);
  m = seg_max(m, group >> 5);
  if (m == 0.0f) m = 1.0f;
  if (publish && j0 % group == 0 && s_group_out) s_group_out[j0 / group] = m;
  return __frcp_rn(m);
}

// Codes of this thread's 32 smoothed values z (positions j0..j0+31 of row trow) given the row's absmax m: alpha =
// fl(m/7), codes rint_even(fl(z * fl(7/m))) clamped to [-8, 7] (R9-R11), packed nibbles (D4 or the decode4
// tiled layout) and / or the GEMM operand bytes; the j0 == 0 thread stores alpha.
RRS_DEVICE void write_codes(const float (&z)[32], float m, int64_t trow, int K, int j0, uint8_t* __restrict__ Xq,
                            int8_t* __restrict__ Xq8, float* __restrict__ scale_out, bool e4m3, bool dec4) {
  float alpha = 1.0f, r = 0.0f;
  if (m > 0.0f) {
    alpha = __fdiv_rn(m, 7.0f);  // stored scale alpha_t = fl(m/7)
    r = __fdiv_rn(7.0f, m);      // R9: codes use fl(7/m)
  }
  if (Xq == nullptr && e4m3) {
    // hot path (rrs_linear): only the E4M3 operand.  rint (RNE) then clamp in f32 -- the same integer as
    // __float2int_rn + clamp -- and one cvt per pair (integers of magnitude <= 8 are exact in E4M3).
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      float q[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)  // R10 round half to even by the 1.5 * 2^23 magic add (exact: |v| < 2^22, and the sum's
        // ulp is 1, so RN picks the even neighbour on a tie) -- two FADDs on the FMA pipe instead of FRND, and x - x
        // gives the canonical +0 for a rounded-to-zero negative (code byte 0x00).  The R11 clamp never binds here:
        // |z| <= m, so |fl(z fl(7/m))| <= 7 (1 + 2^-24)^2 < 7.5 and the rounding gives |q| <= 7
        q[h] = __fsub_rn(__fadd_rn(__fmul_rn(z[k + h], r), 12582912.0f), 12582912.0f);
      uint32_t lo, hi;
      asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\n\tcvt.u32.u16 %0, t;\n\t}"
          : "=r"(lo) : "f"(q[1]), "f"(q[0]));
      asm("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\n\tcvt.u32.u16 %0, t;\n\t}"
          : "=r"(hi) : "f"(q[3]), "f"(q[2]));
      w[k >> 2] = lo | (hi << 16);
    }
    uint4* dst = reinterpret_cast<uint4*>(Xq8 + trow * K + j0);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
  } else {
    uint32_t packed[4] = {0u, 0u, 0u, 0u};
    uint32_t wide[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    int qv[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      int q = __float2int_rn(__fmul_rn(z[k], r));  // R10: round half to even
      q = max(-8, min(7, q));                      // R11
      qv[k] = q;
      wide[k >> 2] |= operand_byte(q, e4m3) << ((k & 3) * 8);
    }
    if (Xq) {
      int64_t off = trow * (K / 2) + j0 / 2;  // D4: row-major [rows][K/2]
      if (dec4) {
        // decode4 layout (rrs.h RRS_W_PACKED4): byte b of the 32-code chunk = q[b] << 4 | q[b + 16] & 0xF; the chunk
        // sits in the contiguous 16 KiB tile (row block of 256, K-block of 128) at row r, slot c ^ ((r >> 1) & 3)
#pragma unroll
        for (int b = 0; b < 16; ++b)
          packed[b >> 2] |= ((uint32_t)((qv[b] & 0xF) << 4) | (uint32_t)(qv[b + 16] & 0xF)) << ((b & 3) * 8);
        const int r = (int)(trow & 255), c = (j0 >> 5) & 3;
        off = (((trow >> 8) * (K >> 7) + (j0 >> 7)) << 14) + r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) packed[k >> 3] |= (uint32_t)(qv[k] & 0xF) << ((k & 7) * 4);  // D4
      }
      *reinterpret_cast<uint4*>(Xq + off) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
    if (Xq8) {
      uint4* dst = reinterpret_cast<uint4*>(Xq8 + trow * K + j0);
      dst[0] = make_uint4(wide[0], wide[1], wide[2], wide[3]);
      dst[1] = make_uint4(wide[4], wide[5], wide[6], wide[7]);
    }
  }
  if (j0 == 0) scale_out[trow] = alpha;
}

// Quantise this thread's 32 positions of one row held in shared memory (xs = the row's f32 values in natural
// column order): Z = X~[perm] * inv_s (Eq. 2, R9), per-token absmax over the TPR threads of the row,
// alpha = fl(m/7), codes rint_even(fl(Z * fl(7/m))) clamped to [-8, 7] (R9-R11), packed nibbles and
// operand bytes.  Contains __syncthreads() when TPR > 32 (every thread of the CTA must call it);
// `after_reads` runs once every thread has finished reading xs (the caller recycles the buffer there).
template <int TPR, class F>
RRS_DEVICE void quant_row(const float* xs, const int (&pj)[32], float inv_s, bool smooth, float* red, int tid, int rr,
                          int64_t trow, int64_t T, int K, int j0, uint8_t* __restrict__ Xq, int8_t* __restrict__ Xq8,
                          float* __restrict__ scale_out, bool e4m3, F after_reads, bool dec4 = false) {
  float z[32];
  float m = 0.0f;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float x = xs[pj[k]];
    z[k] = smooth ? __fmul_rn(x, inv_s) : x;
    m = fmaxf(m, fabsf(z[k]));
  }
  if constexpr (TPR <= 32) {
    m = seg_max(m, TPR);
  } else {
    m = seg_max(m, 32);
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    const int w0 = (rr * TPR) >> 5;
    float mm = 0.0f;
#pragma unroll 4
    for (int w = 0; w < TPR / 32; ++w) mm = fmaxf(mm, red[w0 + w]);
    m = mm;
  }
  __syncthreads();  // every thread has read xs (and red): both may be reused
  after_reads();
  if (trow >= T) return;
  write_codes(z, m, trow, K, j0, Xq, Xq8, scale_out, e4m3, dec4);
}

// ------------------------------------------------------------------------------ a1-a6 fused (prefill, K = 2^m)
//
// One cooperative launch for the whole prologue.  Only s_g reaches the GEMM, and s_g = max over j' in g of
// c_{perm[j']} = max over (t, j' in g) of |X~_{t, perm[j']}| (Eq. 1-2 P:90-91 with the reorder P:106): a max over
// tokens and the group's channels jointly, so this kernel never forms the per-channel c_j (calls that want chan_max
// take the two-kernel path, api.cu):
//   pass 1, per tile of R rows: FWHT (fwht.cuh) -> X~ rounded once to f32 into shared memory (natural column
//     order, over the idle transpose tile) -> each thread gathers its chunk of 32 reordered positions j0..j0+31
//     (perm, through a table of 16-bit shared-memory byte offsets built once per CTA), folds max |X~| into one
//     running maximum (32 | group, so the chunk lies in one group) and stores the 32 values to the workspace in a
//     layout private to this kernel: row t, float4 q < 8 of chunk c at Xr[t K + 4 (q K/32 + c)] (a warp's 16-byte
//     stores are contiguous);
//   group maxima: shared-memory atomicMax per CTA, then one red.max per group per CTA into gmax[G] (library memory);
//   grid barrier (one thread per cluster arrives; the launch is cooperative, so every CTA is resident);
//   pass 2, the same tiles on the same threads (the values are still in L2): s_g (0 -> 1, R8), Z = X~ * fl(1/s_g)
//     (R9), per-token absmax over the row's K/32 threads, codes (write_codes).
// gmax and the barrier counters live in library memory, one slot per call (concurrent calls use different slots),
// zero at module load and reset by the last CTA to leave: no memset launch precedes this kernel.
constexpr int kGroupSlots = 256;
constexpr int kMaxG = 160;  // api.cu kMaxGroups
__device__ unsigned g_group_gmax[kGroupSlots][kMaxG];
__device__ unsigned g_group_bar[kGroupSlots][3];  // [arrive (clusters), depart (CTAs), next row tile (dynamic rows)]
// gmax / barrier slot per call (every prologue that uses the library slots): concurrent calls use different slots
static unsigned next_slot() {
  static std::atomic<unsigned> calls{0};
  return calls.fetch_add(1u, std::memory_order_relaxed) % kGroupSlots;
}

// FWHT plan of the fused kernel: 64 doubles per thread (one transpose per row at K = 4096) where the plan exists
#ifndef RRS_GROUP_B6_MIN_K  // (timeline harness: -DRRS_GROUP_B6_MIN_K=1<<30 builds the 32-double plans everywhere)
#define RRS_GROUP_B6_MIN_K 4096
#endif
template <int K>
struct GroupPlan {
  using P = FwhtPlan<K, (K >= RRS_GROUP_B6_MIN_K ? 6 : 5)>;
};

// CTAs per cluster of the fused prologue: its cluster only aggregates the grid-barrier arrivals (one per cluster).
// Clusters of 4 (which fit on one SM) were measured against 8: the same 568 co-resident CTAs and the same time
// (tools/gpu_r2ap.sh), so the size stays 8.
#ifndef RRS_GROUP_CLUSTER
#define RRS_GROUP_CLUSTER 8
#endif
template <int K>
__host__ __device__ constexpr int group_cluster() { return RRS_GROUP_CLUSTER; }

template <int K>
struct GroupSmem {
  using P = typename GroupPlan<K>::P;
  static constexpr int TPQ = K / 32;                                      // gather chunks per row
  static constexpr int CH = TPQ / P::TP2;                                 // gather chunks per thread
  static constexpr int TILE_D = ((P::TILE_PAD * 8 + 127) / 128) * 128;  // fp64 transposes, then the f32 X~ tile
  static constexpr int STAGE = P::TILE * 2;                             // the bf16 tile (single buffer)
  static constexpr int TBL = P::TILE * 2;                               // 32 u16 offsets per gather chunk
  static constexpr int MAX_TILES = 64;                                  // row tiles a CTA may claim (dynamic rows)
  static constexpr int BYTES = TILE_D + STAGE + TBL + kMaxG * 4 + 2 * 32 * 4 + 32 + MAX_TILES * 8;
  // + gmax, red[2][32], barriers (pass-1 stage, unused, pass-2 ring x 2), the CTA's tile list
  static_assert(2 * P::TILE * 4 <= TILE_D, "pass-2 ring: two f32 tiles over the transpose tile");
  static_assert(P::kPow2 && P::THREADS == P::R * P::TP2 && CH * P::TP2 == TPQ && CH <= 2, "gather chunks");
  // the f32 X~ tile is stored with one pad word per 32 (row stride K + K/32): a reorder that maps a warp's lanes to
  // columns 32 apart (e.g. the identity) would otherwise put all 32 gathers of an instruction in one bank
  static constexpr int KP = K + K / 32;
  static_assert(P::R * KP * 4 <= TILE_D && P::R * KP < 65536, "padded f32 X~ tile overlays the transposes; u16 words");
};

template <int K>
__global__ void __cluster_dims__(group_cluster<K>(), 1, 1)
    __launch_bounds__(GroupPlan<K>::P::THREADS, GroupPlan<K>::P::MIN_BLOCKS)
prologue_group_kernel(const uint16_t* __restrict__ X, int64_t T, float* __restrict__ Xr,
                      const int32_t* __restrict__ perm, float* __restrict__ s_group_out, uint8_t* __restrict__ Xq,
                      int8_t* __restrict__ Xq8, float* __restrict__ scale_out, int e4m3, int group, unsigned slot) {
  using P = typename GroupPlan<K>::P;
  using S = GroupSmem<K>;
  constexpr int TPQ = S::TPQ, CH = S::CH, TP2 = P::TP2;
  extern __shared__ __align__(128) uint8_t smem[];
  double* sm = reinterpret_cast<double*>(smem);
  float* xs = reinterpret_cast<float*>(smem);  // the f32 X~ tile [R][KP], natural order, padded (after the FWHT)
  uint16_t* stage = reinterpret_cast<uint16_t*>(smem + S::TILE_D);
  uint4* tbl = reinterpret_cast<uint4*>(smem + S::TILE_D + S::STAGE);  // [CH][4][THREADS] uint4 = 8 u16 word indices
  unsigned* gmax_sm = reinterpret_cast<unsigned*>(smem + S::TILE_D + S::STAGE + S::TBL);
  float* red = reinterpret_cast<float*>(gmax_sm + kMaxG);
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 2 * 32);
  uint64_t* bar2 = bar + 2;                                 // pass-2 ring (two f32 tiles over the transpose tile)
  int64_t* tiles_sm = reinterpret_cast<int64_t*>(bar + 4);  // [MAX_TILES]: the row tiles this CTA transformed
  unsigned* gmax = g_group_gmax[slot];
  unsigned* gbar = g_group_bar[slot];
  const int tid = threadIdx.x;
  // this thread's gather chunks: row rr of a tile, chunks c = cp + ch TP2 (positions 32 c .. 32 c + 31), ch < CH
  const int rr = tid / TP2, cp = tid % TP2;
  const int G = K / group;
  const int64_t ntiles = (T + P::R - 1) / P::R;

  auto issue = [&](int64_t tile) {
    const int64_t rows = (T - tile * P::R) < P::R ? (T - tile * P::R) : P::R;
    const uint32_t bytes = (uint32_t)(rows * K * 2);
    ptx::mbar_arrive_expect_tx(bar, bytes);
    ptx::bulk_load(stage, X + tile * P::R * K, bytes, bar);
  };
  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::mbar_init(&bar2[0], 1);
    ptx::mbar_init(&bar2[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < ntiles) issue(blockIdx.x);
#pragma unroll
  for (int ch = 0; ch < CH; ++ch) {  // gather table: word index in xs of (row rr, column perm[j0 + k]), two per word
    const int j0 = (cp + ch * TP2) * 32;
    const int4* pp = reinterpret_cast<const int4*>(perm + j0);
    uint32_t w[16];
    auto wi = [&](int c) { return (uint32_t)(rr * S::KP + c + (c >> 5)); };
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int4 p4 = __ldg(pp + q);
      w[2 * q] = wi(p4.x) | (wi(p4.y) << 16);
      w[2 * q + 1] = wi(p4.z) | (wi(p4.w) << 16);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      tbl[(ch * 4 + q) * P::THREADS + tid] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
  for (int g = tid; g < kMaxG; g += P::THREADS) gmax_sm[g] = 0u;
  // (the table and gmax_sm are first read after the FWHT's barriers)

  // ---- pass 1
  // Row tiles: the first is blockIdx.x; later ones are claimed from a counter in library memory (dynamic: a CTA that
  // finishes early takes the next tile, so no CTA runs a whole extra tile behind the rest -- with the static stride
  // 4096 rows over 568 CTAs gave 8 tiles to some and 7 to most), one claim ahead so the atomic's latency is hidden
  // behind a whole tile.  The CTA records its tiles for pass 2.  Very long calls (more claims than the list holds) keep
  // the static stride.
  trace(0, 0);
  constexpr int MT = S::MAX_TILES;
  const bool dyn = ntiles <= (int64_t)(MT / 2) * gridDim.x;
  float gm[CH];
#pragma unroll
  for (int ch = 0; ch < CH; ++ch) gm[ch] = 0.0f;
  int rf, tf;  // (tile row, row-thread) of this thread in the FWHT's last layout
  tile_coords<P>(tid, rf, tf);
  // the X~ stores: out_col(tf, j) = out_col(tf, 0) + out_col(0, j) in disjoint bits (fwht.cuh), so the padded address
  // c + c/32 is a per-thread base plus a compile-time offset per register
  const int c0 = out_col<P>(tf, 0);
  float* xs_row = xs + rf * S::KP + c0 + (c0 >> 5);
  int64_t cur = blockIdx.x, nxt = ntiles;  // (thread 0) this tile and the claimed next one
  if (tid == 0 && cur < ntiles) nxt = dyn ? gridDim.x + (int64_t)atomicAdd(&gbar[2], 1u) : cur + gridDim.x;
  int ntl = 0;
  int64_t tile = blockIdx.x;
  for (int it = 0; tile < ntiles; ++it) {
    int64_t nn = ntiles;  // (thread 0) the tile after nxt, claimed now, used one tile later
    if (tid == 0) {
      tiles_sm[ntl] = cur;
      tiles_sm[ntl + 1] = nxt;  // read by every thread after this tile's barriers
      if (nxt < ntiles) nn = (dyn && ntl + 2 < MT - 1) ? gridDim.x + (int64_t)atomicAdd(&gbar[2], 1u)
                                                        : (dyn ? (int64_t)ntiles : nxt + gridDim.x);
    }
    ptx::mbar_wait(bar, it & 1);
    if (it == 0) trace(0, 1);
    {
      double v[P::E];
      int rr_, tp_;
      fwht_tile<P>(stage, sm, v, rr_, tp_,
                   [&](int j, float f) {
                     const int c = out_col<P>(0, j);
                     xs_row[c + (c >> 5)] = f;
                   },
                   [&] { if (tid == 0 && nxt < ntiles) issue(nxt); });
    }
    __syncthreads();  // the X~ tile is complete
    float z[CH][32];
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 o = tbl[(ch * 4 + q) * P::THREADS + tid];
        const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          z[ch][8 * q + 2 * h] = xs[ow[h] & 0xFFFFu];
          z[ch][8 * q + 2 * h + 1] = xs[ow[h] >> 16];
        }
      }
    const int64_t next_tile = tiles_sm[ntl + 1];
    __syncthreads();  // every gather is done: the tile is rewritten by the next FWHT
    const int64_t trow = tile * P::R + rr;
    if (trow < T) {
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        float4* dst = reinterpret_cast<float4*>(Xr + trow * K) + cp + ch * TP2;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          gm[ch] = fmaxf(gm[ch], fmaxf(fmaxf(fabsf(z[ch][4 * q]), fabsf(z[ch][4 * q + 1])),
                                       fmaxf(fabsf(z[ch][4 * q + 2]), fabsf(z[ch][4 * q + 3]))));
          dst[q * TPQ] = make_float4(z[ch][4 * q], z[ch][4 * q + 1], z[ch][4 * q + 2], z[ch][4 * q + 3]);
        }
      }
    }
    ++ntl;
    tile = next_tile;
    if (tid == 0) {
      cur = nxt;
      nxt = nn;
    }
  }
  // ---- group maxima (values >= +0: unsigned order of the float bits is the float order)
  trace(0, 2);
#pragma unroll
  for (int ch = 0; ch < CH; ++ch) atomicMax(gmax_sm + (cp + ch * TP2) * 32 / group, __float_as_uint(gm[ch]));
  __syncthreads();
  for (int g = tid; g < G; g += P::THREADS)
    if (gmax_sm[g]) atomicMax(gmax + g, gmax_sm[g]);

  // pass 2 reads back this CTA's own pass-1 rows (the same tiles), so the first two are brought into shared memory
  // (two f32 tiles over the idle transpose tile) by bulk copies issued BEFORE the grid barrier: their latency hides
  // behind the barrier wait, and every later tile is fetched two tiles ahead.  Every thread's X~ stores are ordered
  // before the async-proxy reads by its own proxy fence and the CTA barrier that follows.
  float* ring = reinterpret_cast<float*>(smem);
  auto issue2 = [&](int i) {  // tile list entry i -> ring slot i & 1
    const int64_t tile = tiles_sm[i];
    const int64_t rows = (T - tile * P::R) < P::R ? (T - tile * P::R) : P::R;
    const uint32_t bytes = (uint32_t)(rows * K * 4);
    ptx::mbar_arrive_expect_tx(&bar2[i & 1], bytes);
    ptx::bulk_load(ring + (i & 1) * P::TILE, Xr + tile * P::R * K, bytes, &bar2[i & 1]);
  };
  ptx::fence_proxy_async_global();
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < 2 && i < ntl; ++i) issue2(i);

  // ---- grid barrier: the Xr stores and the gmax atomics are visible everywhere
  __threadfence();
  ptx::cluster_sync();
  if (ptx::cluster_ctarank() == 0 && tid == 0) {
    __threadfence();  // (cumulative: orders the whole cluster's stores and atomics before the arrival)
    atomicAdd(&gbar[0], 1u);
    const unsigned nclusters = gridDim.x / group_cluster<K>();
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&gbar[0]) : "memory");
      if (v >= nclusters) break;
    }
  }
  ptx::cluster_sync();
  trace(0, 3);

  // ---- pass 2
  for (int g = tid; g < G; g += P::THREADS) {
    float s = __uint_as_float(__ldcg(gmax + g));
    s = s == 0.0f ? 1.0f : s;  // R8
    reinterpret_cast<float*>(gmax_sm)[g] = s;
    if (blockIdx.x == 0) s_group_out[g] = s;
  }
  __syncthreads();
  float inv_s[CH];
#pragma unroll
  for (int ch = 0; ch < CH; ++ch)  // R9
    inv_s[ch] = __frcp_rn(reinterpret_cast<const float*>(gmax_sm)[(cp + ch * TP2) * 32 / group]);
  if (tid == 0) {  // this CTA has read gmax: the last CTA out resets the slot for a later call
    __threadfence();
    if (atomicAdd(&gbar[1], 1u) == gridDim.x - 1) {
      for (int g = 0; g < G; ++g) gmax[g] = 0u;
      gbar[0] = 0u;
      gbar[1] = 0u;
      gbar[2] = 0u;
    }
  }
  int pr = 0;
  for (int i = 0; i < ntl; ++i, pr ^= 1) {
    const int64_t tile = tiles_sm[i];
    const int64_t trow = tile * P::R + rr;
    const bool live = trow < T;
    ptx::mbar_wait(&bar2[i & 1], (i >> 1) & 1);
    const float4* src = reinterpret_cast<const float4*>(ring + (i & 1) * P::TILE + rr * K);
    float z[CH][32];
    float m = 0.0f;
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x = live ? src[q * TPQ + cp + ch * TP2] : make_float4(0.f, 0.f, 0.f, 0.f);
        z[ch][4 * q] = __fmul_rn(x.x, inv_s[ch]);
        z[ch][4 * q + 1] = __fmul_rn(x.y, inv_s[ch]);
        z[ch][4 * q + 2] = __fmul_rn(x.z, inv_s[ch]);
        z[ch][4 * q + 3] = __fmul_rn(x.w, inv_s[ch]);
        m = fmaxf(m, fmaxf(fmaxf(fabsf(z[ch][4 * q]), fabsf(z[ch][4 * q + 1])),
                           fmaxf(fabsf(z[ch][4 * q + 2]), fabsf(z[ch][4 * q + 3]))));
      }
    }
    __syncthreads();  // every thread has read ring slot i & 1: refill it with tile i + 2
    if (tid == 0 && i + 2 < ntl) issue2(i + 2);
    if constexpr (TP2 <= 32) {
      m = seg_max(m, TP2);
    } else {  // the row's TP2 / 32 warps through red[pr] (double-buffered: one barrier per tile)
      m = seg_max(m, 32);
      float* rb = red + pr * 32;
      if ((tid & 31) == 0) rb[tid >> 5] = m;
      __syncthreads();
      const int w0 = (rr * TP2) >> 5;
      float mm = 0.0f;
#pragma unroll 4
      for (int w = 0; w < TP2 / 32; ++w) mm = fmaxf(mm, rb[w0 + w]);
      m = mm;
    }
    if (live)
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) write_codes(z[ch], m, trow, K, (cp + ch * TP2) * 32, Xq, Xq8, scale_out, e4m3 != 0, false);
  }
  trace(0, 4);
  ptx::pdl_launch_dependents();
}

// ------------------------------------------------------------------------------ a1-a6, decode-sized T
//
// Decode prologue (T <= 64, K = C * 1024, the decode regime of configs[3]): latency, not throughput, decides.  One
// CTA per token row, K/32 threads = C warps:
//   * FWHT: H_K = H_C (x) H_1024 (index i = 1024 a + b) and the butterfly stages commute, so warp c computes output
//     chunk c of the row on its own: v[b] = sum_a (-1)^popcount(a & c) x[1024 a + b] (the H_C mix, read straight from
//     global memory), then FWHT_1024(v) with 5 bits in registers, one warp-private transpose, 5 bits in registers.
//     Every intermediate is a signed subset sum of the row, exact in fp64 under R3; one rounding to f32 gives the
//     correctly rounded X~ (bit-identical to fwht_colmax_kernel).  X~ stays in shared memory.
//   * channel max over all T rows (Eq. 1, R6): CTA 0 zeroes chan_max, grid barrier, one atomicMax per column
//     per row, grid barrier (cooperative launch; barrier counters in library memory, self-cleaning: no memset).
//     T = 1 needs neither: chan_max = |X~| of the single row.
//   * a3-a6 as in the prefill path (quant_row) on the shared-memory row.
// FWHT of one bf16 row xrow[C * 1024] (shared memory) by the C warps of a CTA, each input widened to fp64 once
// (fwht.cuh widen_bf16_hi: `out` receives values in that representation, to be rounded by fwht_round_f32).
// H_K = H_C (x) H_1024 (index i = 1024 a + b); the butterfly stages commute:
//   phase A: warp c transforms chunk c (b bits): 5 bits in registers, a warp-private transpose (tw, 32 x 33), 5 bits;
//            lane l of warp c then holds chunk c at positions 32 j + l (j < 32), stored to y1[1024 c + 32 j + l].
//   phase B: thread tid takes the nb = 32 / C positions b = nb tid .. nb tid + nb - 1 of all C chunks (32 values)
//            and applies H_C across the chunks (a bits); out(i, value) receives every final y[i] exactly once.
// Every intermediate is a signed subset sum of the row: exact in fp64 under R3.  Lane l reads its four 16-byte slots
// of chunk c in the order q ^ rot, rot = (l >> 1) & 3 (a quarter-warp's loads hit 8 distinct bank groups), so
// register k starts with the input at position k ^ m, m = 8 rot; the register butterflies then give
// z[k] = sum_k' (-1)^(k.k') x[k' ^ m] = (-1)^popcount(k & m) y[k], whose sign the transpose store removes (exact).
// Contains __syncthreads (every thread of the CTA must call it).
template <int C, class Out>
RRS_DEVICE void row_fwht_two_level(const uint16_t* xrow, double* tr, double* y1, Out&& out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rot = (lane >> 1) & 3;
  double v[32];
  {  // phase A
    const uint4* src = reinterpret_cast<const uint4*>(xrow + warp * 1024 + lane * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 w = src[q ^ rot];
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // bf16 -> f64, exact (fwht.cuh widen_bf16_hi; `out` rounds with fwht_round_f32)
        v[q * 8 + 2 * h] = widen_bf16_hi(ws[h] << 16);
        v[q * 8 + 2 * h + 1] = widen_bf16_hi(ws[h] & 0xFFFF0000u);
      }
    }
    butterflies<5>(v);
    double* tw = tr + warp * (32 * 33);
#pragma unroll
    for (int e = 0; e < 32; ++e) tw[e * 33 + lane] = (__popc((e >> 3) & rot) & 1) ? -v[e] : v[e];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = tw[lane * 33 + j];
    butterflies<5>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) y1[warp * 1024 + 32 * j + lane] = v[j];
  }
  __syncthreads();
  if constexpr (C == 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) out(32 * j + lane, v[j]);
  } else {  // phase B: v[a * nb + i] = chunk a at position nb tid + i
    constexpr int nb = 32 / C, lg = ilog2_c(C);
    const int b0 = nb * threadIdx.x;
#pragma unroll
    for (int a = 0; a < C; ++a)
#pragma unroll
      for (int i = 0; i < nb; ++i) v[a * nb + i] = y1[a * 1024 + b0 + i];
    // H_C over a: butterflies on the register bits above log2(nb)
#pragma unroll
    for (int hb = 0; hb < lg; ++hb) {
      const int h = nb << hb;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if ((k & h) == 0) {
          const double x0 = v[k], x1 = v[k + h];
          v[k] = x0 + x1;
          v[k + h] = x0 - x1;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < C; ++a)
#pragma unroll
      for (int i = 0; i < nb; ++i) out(a * 1024 + b0 + i, v[a * nb + i]);
  }
}

__device__ unsigned g_small_bar[256][2];  // [slot][arrive, depart]: zero at module load, reset by the last departer

RRS_DEVICE void grid_barrier_selfclean(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&bar[0], 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < nblocks);
    if (atomicAdd(&bar[1], 1u) == nblocks - 1) {  // every block has left the spin: reset for the next use
      bar[0] = 0u;
      bar[1] = 0u;
    }
  }
  __syncthreads();
}

// As above, but the departure count (bar[1]) is left to the caller, which resets the slot after its last read of the
// data the barrier published.
RRS_DEVICE void grid_barrier_selfclean_keep(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&bar[0], 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < nblocks);
  }
  __syncthreads();
}

template <int C>
struct DecodePrologueSmem {
  static constexpr int K = C * 1024;
  static constexpr int TR = C * 32 * 33 * 8;  // warp-private 32 x 32 fp64 transposes (row stride 33); later X~ row f32
  static constexpr int Y1 = K * 8;            // phase-A results (fp64); later chan_max f32
  static constexpr int XB = K * 2;            // the bf16 input row (one bulk copy)
  static constexpr int BYTES = TR + Y1 + XB + 64 * 4 + 16;
  static_assert(TR >= K * 4 && Y1 >= K * 4, "overlays");
};

// One CTA per token row (T <= 64), clusters of up to 8 CTAs (8 rows).  c_j = max over all T rows: the cluster reduces
// its rows through DSMEM (CTA r takes columns [r K/8, (r+1) K/8)) into a per-cluster partial in `scratch`
// ([clusters][K] f32: the workspace's X~ region, unused on this path), one grid barrier (counters in library memory,
// self-cleaning: no memset), then every CTA takes the max over the cluster partials.  T = 1 needs none of it.
template <int C>
__global__ void __launch_bounds__(C * 32)
prologue_decode_kernel(const uint16_t* __restrict__ X, int T, const int32_t* __restrict__ perm,
                       unsigned* __restrict__ chan_max_bits, float* __restrict__ scratch, float* __restrict__ s_group_out,
                       uint8_t* __restrict__ Xq, int8_t* __restrict__ Xq8, float* __restrict__ scale_out, int e4m3,
                       int group, unsigned* __restrict__ bar) {
  constexpr int K = C * 1024, TPR = K / 32;
  using S = DecodePrologueSmem<C>;
  extern __shared__ __align__(128) uint8_t smem[];
  double* tr = reinterpret_cast<double*>(smem);
  double* y1 = reinterpret_cast<double*>(smem + S::TR);
  float* xs = reinterpret_cast<float*>(smem);          // X~ row (natural column order), after phase A
  float* cms = reinterpret_cast<float*>(smem + S::TR);  // chan_max, after phase B
  uint16_t* xrow = reinterpret_cast<uint16_t*>(smem + S::TR + S::Y1);
  float* red = reinterpret_cast<float*>(smem + S::TR + S::Y1 + S::XB);
  uint64_t* bar_x = reinterpret_cast<uint64_t*>(smem + S::TR + S::Y1 + S::XB + 64 * 4);
  ptx::pdl_launch_dependents();  // the decode GEMM may get resident (and start its W stream) on the SMs left free
  const int tid = threadIdx.x;
  const int t = blockIdx.x;
  const bool live = t < T;  // the grid is padded to whole clusters
  const int j0 = tid * 32;
  if (tid == 0) {  // the whole bf16 row in one bulk copy
    ptx::mbar_init(bar_x, 1);
    ptx::fence_barrier_init();
    if (live) {
      ptx::mbar_arrive_expect_tx(bar_x, S::XB);
      ptx::bulk_load(xrow, X + (int64_t)t * K, S::XB, bar_x);
    }
  }
  trace(2, 0);
  int pj[32];
  load_perm32(perm, j0, pj);  // an offline input
  __syncthreads();
  if (live) ptx::mbar_wait(bar_x, 0);
  else
    for (int i = tid; i < K / 2; i += TPR) reinterpret_cast<uint32_t*>(xrow)[i] = 0u;  // a zero row: |X~| = 0
  __syncthreads();
  trace(2, 1);
  // ---- a1 (X~ rounded once to f32, natural column order, into xs over the idle transposes)
  row_fwht_two_level<C>(xrow, tr, y1, [&](int i, double d) { xs[i] = fwht_round_f32(d); });
  __syncthreads();
  trace(2, 2);
  // ---- a2: c_j = max over all T rows
  if (gridDim.x > 1) {
    // (1) cluster max over its 8 rows: CTA r reduces columns [r K/8, (r+1) K/8) (one float4 of 4 columns per thread
    //     and peer, all 8 DSMEM loads in flight) into the cluster partial in scratch
    ptx::cluster_sync();  // every CTA's xs is complete
    trace(2, 3);
    const uint32_t rank = ptx::cluster_ctarank();
    constexpr int SL = K / 8;                // columns per rank
    static_assert(SL / 4 <= TPR, "one float4 per thread");
    const int ncl = (int)(gridDim.x / 8);
    const int col4 = (int)rank * SL + 4 * tid;  // this thread's 4 columns (tid < SL / 4)
    if (tid < SL / 4) {
      float4 v[8];
#pragma unroll
      for (uint32_t r = 0; r < 8; ++r) v[r] = ptx::ld_dsmem_f32x4(xs + col4, r);
      float4 m = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        m.x = fmaxf(m.x, fabsf(v[r].x)); m.y = fmaxf(m.y, fabsf(v[r].y));
        m.z = fmaxf(m.z, fabsf(v[r].z)); m.w = fmaxf(m.w, fabsf(v[r].w));
      }
      *reinterpret_cast<float4*>(scratch + (int64_t)(blockIdx.x / 8) * K + col4) = m;
    }
    trace(2, 7);
    // (the grid barrier's fence in thread 0, after the CTA barrier, releases every thread's scratch stores; no peer
    // ever writes xs, and the cluster barrier in (3) keeps every CTA alive until its peers' DSMEM reads are done)
    grid_barrier_selfclean(bar, gridDim.x);
    trace(2, 9);
    // (2) the same slice over all clusters (ncl float4 loads in flight per thread), into this CTA's cms slice
    if (tid < SL / 4) {
      float4 m = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      for (int q0 = 0; q0 < ncl; q0 += 8) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          v[q] = q0 + q < ncl ? __ldcg(reinterpret_cast<const float4*>(scratch + (int64_t)(q0 + q) * K + col4))
                              : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          m.x = fmaxf(m.x, v[q].x); m.y = fmaxf(m.y, v[q].y); m.z = fmaxf(m.z, v[q].z); m.w = fmaxf(m.w, v[q].w);
        }
      }
      *reinterpret_cast<float4*>(cms + col4) = m;
      if (blockIdx.x < 8) *reinterpret_cast<float4*>(chan_max_bits + col4) = m;  // float bits (>= +0)
    }
    // (3) every CTA gathers the other seven slices from its cluster peers (all 8 loads in flight, then the stores)
    trace(2, 10);
    ptx::cluster_sync();
    trace(2, 11);
    {
      constexpr int PER = K / 4 / TPR;  // 8 float4 per thread
      float4 g[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = tid + k * TPR;
        const uint32_t r = (uint32_t)(4 * i / SL);
        g[k] = r != rank ? ptx::ld_dsmem_f32x4(cms + 4 * i, r) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int i = tid + k * TPR;
        if ((uint32_t)(4 * i / SL) != rank) *reinterpret_cast<float4*>(cms + 4 * i) = g[k];
      }
    }
    ptx::cluster_sync();  // no CTA exits (or overwrites cms) while a peer still reads it
  } else {
    for (int i = tid; i < K; i += TPR) {
      cms[i] = fabsf(xs[i]);
      chan_max_bits[i] = __float_as_uint(cms[i]);
    }
  }
  __syncthreads();
  trace(2, 4);
  // ---- a3-a6 on this CTA's row
  const float inv_s = group_inv_scale(cms, pj, j0, blockIdx.x == 0, s_group_out, group);
  trace(2, 5);
  if (live) quant_row<TPR>(xs, pj, inv_s, true, red, tid, 0, t, T, K, j0, Xq, Xq8, scale_out, e4m3 != 0, [] {});
  trace(2, 6);
}

// The decode prologue without a chan_max output (the rrs_linear hot path).  s_g = max over (t, j' in g) of |X~_{t,perm[j']}|
// (Eq. 1-2 P:90-91 with the reorder P:106) is a joint max over tokens and the group's channels, so the CTAs never form
// c_j: each CTA gathers its row in reordered order, reduces its group maxima over the group's L/32 lanes and folds them
// into gmax[G] (library memory, one red.max per group per CTA); one grid barrier; every thread reads its group's s_g.
// T = 1 needs no barrier at all (the row's group maxima are s_g).  gmax and the barrier counters are per-call slots,
// zero at module load and reset by the last CTA to leave (no memset launch).
template <int C>
__global__ void __launch_bounds__(C * 32)
prologue_decode_group_kernel(const uint16_t* __restrict__ X, const int32_t* __restrict__ perm,
                             float* __restrict__ s_group_out, uint8_t* __restrict__ Xq, int8_t* __restrict__ Xq8,
                             float* __restrict__ scale_out, int e4m3, int group, unsigned slot) {
  constexpr int K = C * 1024, TPR = K / 32;
  using S = DecodePrologueSmem<C>;
  extern __shared__ __align__(128) uint8_t smem[];
  double* tr = reinterpret_cast<double*>(smem);
  double* y1 = reinterpret_cast<double*>(smem + S::TR);
  float* xs = reinterpret_cast<float*>(smem);  // X~ row (natural column order), after phase A
  uint16_t* xrow = reinterpret_cast<uint16_t*>(smem + S::TR + S::Y1);
  float* red = reinterpret_cast<float*>(smem + S::TR + S::Y1 + S::XB);
  uint64_t* bar_x = reinterpret_cast<uint64_t*>(smem + S::TR + S::Y1 + S::XB + 64 * 4);
  ptx::pdl_launch_dependents();  // the decode GEMM may get resident (and start its W stream) on the SMs left free
  const int tid = threadIdx.x;
  const int t = blockIdx.x;
  const int j0 = tid * 32;
  if (tid == 0) {  // the whole bf16 row in one bulk copy
    ptx::mbar_init(bar_x, 1);
    ptx::fence_barrier_init();
    ptx::mbar_arrive_expect_tx(bar_x, S::XB);
    ptx::bulk_load(xrow, X + (int64_t)t * K, S::XB, bar_x);
  }
  trace(2, 0);
  int pj[32];
  load_perm32(perm, j0, pj);  // an offline input
#pragma unroll
  for (int k = 0; k < 32; ++k) pj[k] += pj[k] >> 5;  // xs keeps one pad word per 32 columns (no bank-aligned gathers)
  __syncthreads();
  ptx::mbar_wait(bar_x, 0);
  trace(2, 1);
  // ---- a1 (X~ rounded once to f32, natural column order, padded, into xs over the idle transposes)
  row_fwht_two_level<C>(xrow, tr, y1, [&](int i, double d) { xs[i + (i >> 5)] = fwht_round_f32(d); });
  __syncthreads();
  trace(2, 2);
  // ---- a2 + a4: this row's maximum over each group of reordered positions (32 | group: a thread's chunk is in one group)
  float m = 0.0f;
#pragma unroll
  for (int k = 0; k < 32; ++k) m = fmaxf(m, fabsf(xs[pj[k]]));
  m = seg_max(m, group >> 5);
  const int g = j0 / group;
  if (gridDim.x > 1) {
    unsigned* gmax = g_group_gmax[slot];
    unsigned* gbar = g_group_bar[slot];
    if (j0 % group == 0) atomicMax(gmax + g, __float_as_uint(m));  // float bits of values >= +0
    grid_barrier_selfclean_keep(gbar, gridDim.x);
    trace(2, 3);
    m = __uint_as_float(__ldcg(gmax + g));
    __syncthreads();  // every thread of this CTA has read gmax
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(&gbar[1], 1u) == gridDim.x - 1) {  // the last CTA to leave resets the slot for a later call
        for (int i = 0; i < K / group; ++i) gmax[i] = 0u;
        gbar[0] = 0u;
        gbar[1] = 0u;
      }
    }
  }
  if (m == 0.0f) m = 1.0f;  // R8
  if (blockIdx.x == 0 && j0 % group == 0) s_group_out[g] = m;
  trace(2, 4);
  // ---- a3, a5, a6 on this CTA's row
  quant_row<TPR>(xs, pj, __frcp_rn(m), true, red, tid, 0, t, gridDim.x, K, j0, Xq, Xq8, scale_out, e4m3 != 0, [] {});
  trace(2, 6);
}

template <int C>
static cudaError_t launch_decode_group_k(const uint16_t* X, int64_t T, const int32_t* perm, float* s_group, uint8_t* Xq,
                                         int8_t* Xq8, float* scale, bool e4m3, int group, unsigned slot, cudaStream_t st) {
  auto kern = prologue_decode_group_kernel<C>;
  constexpr int smem = DecodePrologueSmem<C>::BYTES;
  cudaError_t e = prepare_kernel(kern, smem, C * 32);
  if (e != cudaSuccess) return e;
  int ei = (int)e4m3;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)T);
  cfg.blockDim = dim3(C * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = T > 1 ? 1 : 0;  // a single row needs no barrier
  return cudaLaunchKernelEx(&cfg, kern, X, perm, s_group, Xq, Xq8, scale, ei, group, slot);
}

template <int C>
static cudaError_t launch_decode_prologue_k(const uint16_t* X, int64_t T, const int32_t* perm, unsigned* cm,
                                            float* scratch, float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale,
                                            bool e4m3, int group, unsigned slot, cudaStream_t st) {
  if (cm == nullptr) return launch_decode_group_k<C>(X, T, perm, s_group, Xq, Xq8, scale, e4m3, group, slot, st);
  auto kern = prologue_decode_kernel<C>;
  constexpr int smem = DecodePrologueSmem<C>::BYTES;
  cudaError_t e = prepare_kernel(kern, smem, C * 32);
  if (e != cudaSuccess) return e;
  void* bar = nullptr;
  e = cudaGetSymbolAddress(&bar, g_small_bar);
  if (e != cudaSuccess) return e;
  unsigned* b = static_cast<unsigned*>(bar) + 2 * (slot & 255u);
  int Ti = (int)T, ei = (int)e4m3;
  const unsigned grid = T == 1 ? 1u : (unsigned)((T + 7) / 8 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 8;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = grid > 1 ? 2 : 0;  // a single row needs neither (no barrier, no cluster)
  return cudaLaunchKernelEx(&cfg, kern, X, Ti, perm, cm, scratch, s_group, Xq, Xq8, scale, ei, group, b);
}

bool prologue_decode_supports(int64_t T, int64_t K, int group) {
  return T >= 1 && T <= 64 && K >= 1024 && K <= 8192 && (K & (K - 1)) == 0 && group >= 32;
}

cudaError_t launch_prologue_decode(const uint16_t* X, int64_t T, int64_t K, const int32_t* perm, unsigned* chan_max_bits,
                                   float* scratch, float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3,
                                   int group, cudaStream_t st) {
  const unsigned slot = next_slot();
  switch (K) {
#define RRS_CASE(c) case c * 1024: return launch_decode_prologue_k<c>(X, T, perm, chan_max_bits, scratch, s_group, Xq, Xq8, scale, e4m3, group, slot, st);
    RRS_CASE(1) RRS_CASE(2) RRS_CASE(4) RRS_CASE(8)
#undef RRS_CASE
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------ a2 without a1 (variants)
// RRS_NO_ROTATION / RRS_PREROTATED (rrs.h): X~ = X exactly (bf16 -> f32), plus the runtime channel max when
// chan_max_bits != nullptr (Eq. 1): column j of a row slab per thread, one atomicMax per column per CTA.
__global__ void __launch_bounds__(256)
convert_colmax_kernel(const uint16_t* __restrict__ X, int64_t T, int K, int64_t rows_per, float* __restrict__ Xr,
                      unsigned* __restrict__ chan_max_bits) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= K) return;
  const int64_t t0 = blockIdx.y * rows_per, t1 = t0 + rows_per < T ? t0 + rows_per : T;
  float m = 0.0f;
  for (int64_t t = t0; t < t1; ++t) {
    const float x = __uint_as_float((uint32_t)__ldg(X + t * K + j) << 16);
    Xr[t * K + j] = x;
    m = fmaxf(m, fabsf(x));
  }
  if (chan_max_bits && t1 > t0) atomicMax(chan_max_bits + j, __float_as_uint(m));
}

cudaError_t launch_convert_colmax(const uint16_t* X, int64_t T, int64_t K, unsigned* chan_max_bits, float* Xr, int nsm,
                                  cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  const int cols = (int)((K + 255) / 256);
  const int64_t slabs = std::max<int64_t>(1, std::min<int64_t>(T, (4LL * nsm + cols - 1) / cols));
  const int64_t rows_per = (T + slabs - 1) / slabs;
  convert_colmax_kernel<<<dim3(cols, (unsigned)((T + rows_per - 1) / rows_per)), 256, 0, st>>>(X, T, (int)K, rows_per,
                                                                                               Xr, chan_max_bits);
  return cudaGetLastError();
}

template <int K>
struct QuantPlan {
  static constexpr int TPR = K / 32;                                       // threads per row, 32 codes each
  static constexpr int R = TPR >= 256 ? 1 : 256 / TPR;                     // rows per CTA tile (8 warps)
  static constexpr int THREADS = R * TPR;
  static constexpr int TILE = R * K;                                       // f32 elements per tile
  // TMA-bulk ring deep enough to cover the load latency (2 CTAs/SM up to K = 8192, 1 CTA/SM beyond);
  // chan_max is staged in the first ring slot before any row load is issued
  static constexpr int BUDGET = K <= 8192 ? 96 * 1024 : 160 * 1024;
  static constexpr int STAGES = min_c(8, max_c(2, BUDGET / (TILE * 4)));
  static constexpr int BYTES = STAGES * TILE * 4 + K * 4 + 64 * 4 + 8 * 8 + 64;  // ring + chan_max + red + bars
  static_assert(THREADS <= 1024 && THREADS % 32 == 0, "quant layout");
};

template <int K>
__global__ void __launch_bounds__(QuantPlan<K>::THREADS)
smooth_quant_kernel(const float* __restrict__ Xr, int64_t T, const int32_t* __restrict__ perm,
                    const unsigned* __restrict__ chan_max_bits, float* __restrict__ s_group_out,
                    uint8_t* __restrict__ Xq, int8_t* __restrict__ Xq8, float* __restrict__ scale_out, int e4m3,
                    int group, int dec4) {
  using Q = QuantPlan<K>;
  constexpr int TPR = Q::TPR;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int STAGES = Q::STAGES;
  float* stage = reinterpret_cast<float*>(smem);
  float* cms = reinterpret_cast<float*>(smem + STAGES * Q::TILE * 4);   // chan_max [K]
  float* red = cms + K;
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 64);
  const int tid = threadIdx.x;
  const int rr = tid / TPR;                 // tile row of this thread
  const int j0 = (tid % TPR) * 32;          // first reordered position j'
  const int64_t ntiles = (T + Q::R - 1) / Q::R;
  const bool smooth = chan_max_bits != nullptr;

  // tiles are visited in REVERSE order: the rotate pass wrote the highest rows last, so when X~ is larger than L2
  // (C3 down: 235 MB) its most recently written part is still in L2 when this pass starts
  auto phys = [&](int64_t li) { return ntiles - 1 - li; };
  auto issue = [&](int64_t li, int buf) {
    const int64_t tile = phys(li);
    const int64_t rows = (T - tile * Q::R) < Q::R ? (T - tile * Q::R) : Q::R;
    const uint32_t bytes = (uint32_t)(rows * K * 4);
    ptx::mbar_arrive_expect_tx(&bar[buf], bytes);
    ptx::bulk_load(stage + buf * Q::TILE, Xr + tile * Q::R * K, bytes, &bar[buf]);
  };
  trace(1, 2);
  if (tid == 0) {
    for (int b = 0; b < STAGES; ++b) ptx::mbar_init(&bar[b], 1);
    ptx::fence_barrier_init();
  }
  trace(1, 0);
  int pj[32];  // perm is an offline input: read it before waiting for the FWHT pass
  load_perm32(perm, j0, pj);
  ptx::pdl_launch_dependents();  // the GEMM may get resident (and start its W stream) on SMs we leave free
  ptx::pdl_wait();  // X~ and chan_max come from fwht_colmax_kernel / prologue_small_kernel
  __syncthreads();
  trace(1, 1);
  if (tid == 0) {  // start the row loads first; the s_g setup below overlaps them
    for (int b = 0; b < STAGES; ++b)
      if (blockIdx.x + (int64_t)b * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)b * gridDim.x, b);
  }
  float inv_s = 1.0f;
  if (smooth) {
    for (int c = tid * 4; c < K; c += Q::THREADS * 4)  // chan_max -> shared memory, coalesced
      *reinterpret_cast<uint4*>(cms + c) = __ldcg(reinterpret_cast<const uint4*>(chan_max_bits + c));
    __syncthreads();
    inv_s = group_inv_scale(cms, pj, j0, blockIdx.x == 0 && rr == 0, s_group_out, group);
  } else if (s_group_out && blockIdx.x == 0) {
    for (int g = tid; g < K / group; g += Q::THREADS) s_group_out[g] = 1.0f;  // RRS_NO_SMOOTH baseline: s_g = 1
  }
  trace(1, 2);

  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it % STAGES;
    ptx::mbar_wait(&bar[buf], (it / STAGES) & 1);
    trace(1, 3 + (it < 10 ? it : 10));
    quant_row<TPR>(stage + buf * Q::TILE + rr * K, pj, inv_s, smooth, red, tid, rr, phys(tile) * Q::R + rr, T, K, j0, Xq,
                   Xq8, scale_out, e4m3 != 0, [&] {
                     if (tid == 0 && tile + STAGES * (int64_t)gridDim.x < ntiles)
                       issue(tile + STAGES * (int64_t)gridDim.x, buf);
                   }, dec4 != 0);
  }
  trace(1, 15);
  ptx::pdl_launch_dependents();
}

// perm[rank(j)] = j, rank by (c descending, index ascending)  -- R5 / R21
__global__ void perm_rank_kernel(const float* __restrict__ c, int K, int32_t* __restrict__ perm) {
  extern __shared__ float cs[];
  for (int i = threadIdx.x; i < K; i += blockDim.x) cs[i] = c[i];
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  const float cj = cs[j];
  int rank = 0;
  for (int i = 0; i < K; ++i) {
    const float ci = cs[i];
    rank += (ci > cj) || (ci == cj && i < j);
  }
  perm[rank] = j;
}

// ------------------------------------------------------------------------------- host launchers

template <class F>
static int grid_for(F kern, int threads, int smem, int64_t tiles, int nsm) {
  int per_sm = 1;
  prepare_kernel(kern, smem, threads, &per_sm);
  return (int)std::min<int64_t>(tiles, (int64_t)nsm * per_sm);
}

template <int K>
static cudaError_t launch_colmax_k(const uint16_t* X, int64_t T, unsigned* cm, float* Xr, int nsm,
                                   cudaStream_t st) {
  using P = FwhtPlan<K>;
  auto kern = fwht_colmax_kernel<K>;
  const int smem = ColmaxSmem<K>::BYTES;
  cudaError_t e = prepare_kernel(kern, smem, P::THREADS);
  if (e != cudaSuccess) return e;
  // persistent: only as many clusters as can be co-resident (a cluster of 8 must fit in one GPC, so this is
  // below SMs x CTAs-per-SM / 8); late clusters would otherwise run as a second wave
  int max_clusters = max_active_clusters(kern, colmax_cluster<K>(), P::THREADS, smem);
  if (max_clusters < 1) max_clusters = nsm / colmax_cluster<K>();
  const int64_t tiles = (T + P::R - 1) / P::R;
  if (tiles == 0) return cudaSuccess;
  const int64_t clusters = std::min<int64_t>(max_clusters, (tiles + colmax_cluster<K>() - 1) / colmax_cluster<K>());
  const int grid = (int)clusters * colmax_cluster<K>();  // whole clusters (CTAs without a tile are fine)
  kern<<<grid, P::THREADS, smem, st>>>(X, T, cm, Xr);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_group_k(const uint16_t* X, int64_t T, float* Xr, const int32_t* perm, float* s_group,
                                  uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3, int group, unsigned slot,
                                  cudaStream_t st) {
  using P = typename GroupPlan<K>::P;
  auto kern = prologue_group_kernel<K>;
  const int smem = GroupSmem<K>::BYTES;
  cudaError_t e = prepare_kernel(kern, smem, P::THREADS);
  if (e != cudaSuccess) return e;
  // every CTA must be resident at once (grid barrier): the grid is at most the co-resident cluster count, and the
  // launch is COOPERATIVE, so the runtime refuses it (instead of letting it hang) when the grid cannot be co-resident;
  // the caller then falls back to the two-kernel prologue
  const int max_clusters = max_active_clusters(kern, group_cluster<K>(), P::THREADS, smem);
  if (max_clusters < 1) return cudaErrorCooperativeLaunchTooLarge;
  const int64_t tiles = (T + P::R - 1) / P::R;
  const int64_t clusters =
      std::max<int64_t>(1, std::min<int64_t>(max_clusters, (tiles + group_cluster<K>() - 1) / group_cluster<K>()));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * group_cluster<K>()));
  cfg.blockDim = dim3(P::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, X, T, Xr, perm, s_group, Xq, Xq8, scale, (int)e4m3, group, slot);
}

template <int K>
static cudaError_t launch_quant_k(const float* Xr, int64_t T, const int32_t* perm, const unsigned* cm,
                                  float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3, int group, int nsm,
                                  cudaStream_t st, bool dec4) {
  using Q = QuantPlan<K>;
  auto kern = smooth_quant_kernel<K>;
  cudaError_t e = prepare_kernel(kern, Q::BYTES, Q::THREADS);
  if (e != cudaSuccess) return e;
  // persistent: at most 2 CTAs per SM, so the per-CTA setup (chan_max load, s_g) is amortised over many rows
  int grid = (int)std::min<int64_t>(grid_for(kern, Q::THREADS, Q::BYTES, (T + Q::R - 1) / Q::R, nsm), 2 * nsm);
  if (grid == 0) {
    if (cm == nullptr || s_group == nullptr) return cudaSuccess;
    grid = 1;  // T == 0: still publish s_group (all ones, R8)
  }
  return launch_pdl(kern, grid, Q::THREADS, Q::BYTES, st, Xr, T, perm, cm, s_group, Xq, Xq8, scale, (int)e4m3, group,
                    (int)dec4);
}

#define RRS_FOR_EACH_K(M) M(128) M(256) M(512) M(1024) M(2048) M(4096) M(8192) M(16384) M(7168) M(14336)

#define RRS_FOR_EACH_POW2_K(M) M(128) M(256) M(512) M(1024) M(2048) M(4096) M(8192) M(16384)

bool prologue_fused_supports_k(int64_t K) { return K >= 128 && K <= 16384 && (K & (K - 1)) == 0; }

cudaError_t launch_prologue_fused(const uint16_t* X, int64_t T, int64_t K, float* Xr, const int32_t* perm,
                                  float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3, int group,
                                  cudaStream_t st) {
  if (K / group > kMaxG) return cudaErrorInvalidValue;
  const unsigned slot = next_slot();
  switch (K) {
#define RRS_CASE(k) case k: return launch_group_k<k>(X, T, Xr, perm, s_group, Xq, Xq8, scale, e4m3, group, slot, st);
    RRS_FOR_EACH_POW2_K(RRS_CASE)
#undef RRS_CASE
    default: return cudaErrorInvalidValue;
  }
}

bool prologue_supports_k(int64_t K) {
  switch (K) {
#define RRS_CASE(k) case k: return true;
    RRS_FOR_EACH_K(RRS_CASE)
#undef RRS_CASE
    default: return false;
  }
}

cudaError_t launch_fwht_colmax(const uint16_t* X, int64_t T, int64_t K, unsigned* chan_max_bits, float* Xr,
                               int nsm, cudaStream_t st) {
  switch (K) {
#define RRS_CASE(k) case k: return launch_colmax_k<k>(X, T, chan_max_bits, Xr, nsm, st);
    RRS_FOR_EACH_K(RRS_CASE)
#undef RRS_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_smooth_quant(const float* Xr, int64_t T, int64_t K, const int32_t* perm,
                                const unsigned* chan_max_bits, float* s_group, uint8_t* Xq, int8_t* Xq8,
                                float* scale, bool e4m3, int group, int nsm, cudaStream_t st, bool dec4) {
  switch (K) {
#define RRS_CASE(k) case k: return launch_quant_k<k>(Xr, T, perm, chan_max_bits, s_group, Xq, Xq8, scale, e4m3, group, nsm, st, dec4);
    RRS_FOR_EACH_K(RRS_CASE)
#undef RRS_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_perm_rank(const float* c, int64_t K, int32_t* perm, cudaStream_t st) {
  const int threads = 256;
  const int blocks = (int)((K + threads - 1) / threads);
  const size_t smem = (size_t)K * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(perm_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  perm_rank_kernel<<<blocks, threads, smem, st>>>(c, (int)K, perm);
  return cudaGetLastError();
}

}  // namespace rrs

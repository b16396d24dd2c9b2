// RRS fused grouped GEMM on tcgen05, sm_100a.
//
//   P_g[t][n] = sum_{j' in group g} Xq8[t][j'] * Wq8[n][j']          (fig:framework (3) P:103)
//   Y[t][n]   = out_scale * alpha_t * beta_n * sum_g s_g * f32(P_g)   ("the runtime smoothing scales are
//                                                                     applied to the dequantized interim
//                                                                     result"; R14, R15)
//
// Design: persistent, one CTA per SM, 320 threads = 10 warps:
//   warp 0      TMA producer: 128x128 int8 X tile + 256x128 int8 W tile per group into a 4-stage
//               SMEM ring (SWIZZLE_128B: one 128-code group is exactly one 128-byte swizzle row);
//   warp 1      TMEM allocator + single-thread tcgen05.mma.kind::i8 issuer (M=128, N=256, K=32, 4 per
//               group) into one of two 256-column int32 TMEM accumulators, alternating per group;
//   warps 2-9   promotion/epilogue: tcgen05.ld the group's int32 partials (lane quadrant = warp % 4,
//               column half = (warp-2)/4), convert exactly with the 1.5*2^23 magic bias (|P_g| <= 6272
//               < 2^22), acc = fma(s_g, P_g, acc) in registers, release the TMEM buffer, and after the
//               last group scale by alpha_t * beta_n * out_scale and store Y.
// The MMA of group g+1 overlaps the promotion of group g (two TMEM buffers).  In plain mode (the
// per-channel A4W4 baseline of P:322) the MMA accumulates all K into one buffer per tile instead.
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace rrs {

namespace gemm {
constexpr int BM = 128;        // tokens per tile   (TMEM lanes)
constexpr int BN = 256;        // outputs per tile  (TMEM columns per accumulator)
constexpr int BK = 128;        // one smoothing group = one GEMM K-block
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;          // 16 KiB
constexpr int B_BYTES = BN * BK;          // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_EPI_WARPS = 8;
constexpr int THREADS = 64 + NUM_EPI_WARPS * 32;
constexpr int MAX_G = 128;                 // K <= 16384
constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 1024 /*barriers, scales*/ +
                           MAX_G * 4 + BN * 4;
}  // namespace gemm

struct GemmParams {
  const float* x_scale;
  const float* s_group;
  const float* w_scale;
  int T, N, K, G;
  int num_m, num_n, num_tiles;
  float out_scale;
  void* Y;
  int64_t ldy;
  int32_t* P_debug;
};

template <bool kPlain, bool kF32Out>
__global__ void __launch_bounds__(gemm::THREADS, 1)
rrs_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                GemmParams p) {
  using namespace gemm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* taddr_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* s_sm = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 1024);
  float* beta_sm = s_sm + MAX_G;

  const uint32_t warp = ptx::warp_idx();
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_w);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], NUM_EPI_WARPS);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(taddr_slot, 512);
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
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int m_blk = tile % p.num_m, n_blk = tile / p.num_m;
        for (int kb = 0; kb < p.G; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          ptx::tma_load_2d(sA + stage * A_BYTES, &tmap_x, &full[stage], kb * BK, m_blk * BM, ptx::kEvictNormal);
          ptx::tma_load_2d(sB + stage * B_BYTES, &tmap_w, &full[stage], kb * BK, n_blk * BN, ptx::kEvictNormal);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc_iter = 0;  // number of accumulator buffers filled so far
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < p.G; ++kb) {
        const uint32_t b = acc_iter & 1;
        if (kPlain ? kb == 0 : true) {
          ptx::mbar_wait(&tempty[b], ((acc_iter >> 1) & 1) ^ 1);
        }
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t a_desc = ptx::smem_desc_sw128(sA + stage * A_BYTES);
          const uint64_t b_desc = ptx::smem_desc_sw128(sB + stage * B_BYTES);
          const uint32_t d = tmem_base + b * BN;
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            // advance 32 bytes (= 32 int8 codes) along K inside the 128-byte swizzle row
            const uint32_t acc = kPlain ? (kb > 0 || k > 0) : (k > 0);
            ptx::mma_i8(d, a_desc + 2 * k, b_desc + 2 * k, idesc, acc);
          }
          ptx::mma_commit(&empty[stage]);
          if (!kPlain || kb == p.G - 1) ptx::mma_commit(&tfull[b]);
        }
        __syncwarp();
        if (!kPlain || kb == p.G - 1) ++acc_iter;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------------ promotion + epilogue
    const int ew = warp - 2;                 // 0..7
    const int quad = warp & 3;               // TMEM lane quadrant this warp may access
    const int half = ew >> 2;                // column half of the 256-wide tile
    const int row_in_tile = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint32_t acc_iter = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const int m_blk = tile % p.num_m, n_blk = tile / p.num_m;
      const int row = m_blk * BM + row_in_tile;
      const int col0 = n_blk * BN + half * 128;
      // stage beta for this tile (named barrier among the 256 epilogue threads)
      asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32));
      if (p.w_scale) {
        const int c = threadIdx.x - 64;
        const int n = n_blk * BN + c;
        beta_sm[c] = (n < p.N) ? p.w_scale[n] : 0.0f;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32));

      float acc[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) acc[c] = 0.0f;
      const int ngroups = kPlain ? 1 : p.G;
      for (int g = 0; g < ngroups; ++g) {
        const uint32_t b = acc_iter & 1;
        ptx::mbar_wait(&tfull[b], (acc_iter >> 1) & 1);
        ptx::tc_fence_after();
        const float s = kPlain ? 1.0f : s_sm[g];
        const uint32_t tbase = tmem_base + lane_off + b * BN + half * 128;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          RRS_TMEM_LD32(tbase + cc * 32, r);
          ptx::tmem_ld_wait();
          if (p.P_debug != nullptr && row < p.T) {
            const int gg = kPlain ? 0 : g;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = col0 + cc * 32 + j;
              if (n < p.N) p.P_debug[((int64_t)gg * p.T + row) * p.N + n] = (int32_t)r[j];
            }
          }
          if (kPlain) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[cc * 32 + j] = (float)(int32_t)r[j];  // exact: |sum| < 2^24
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              // exact int32 -> f32 for |P| < 2^22: bits(1.5*2^23 + P) - 1.5*2^23
              const float f = __uint_as_float(r[j] + 0x4B400000u) - 12582912.0f;
              acc[cc * 32 + j] = fmaf(s, f, acc[cc * 32 + j]);
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty[b]);
        ++acc_iter;
      }
      // ---- epilogue: Y = acc * (alpha_t * out_scale) * beta_n
      if (p.Y != nullptr && row < p.T) {
        const float rs = p.x_scale[row] * p.out_scale;
        if constexpr (kF32Out) {
          float* yrow = reinterpret_cast<float*>(p.Y) + (int64_t)row * p.ldy;
#pragma unroll
          for (int c = 0; c < 128; c += 4) {
            const int n = col0 + c;
            float4 v;
            v.x = (acc[c] * rs) * beta_sm[half * 128 + c];
            v.y = (acc[c + 1] * rs) * beta_sm[half * 128 + c + 1];
            v.z = (acc[c + 2] * rs) * beta_sm[half * 128 + c + 2];
            v.w = (acc[c + 3] * rs) * beta_sm[half * 128 + c + 3];
            if (n + 3 < p.N) {
              *reinterpret_cast<float4*>(yrow + n) = v;
            } else {
              if (n < p.N) yrow[n] = v.x;
              if (n + 1 < p.N) yrow[n + 1] = v.y;
              if (n + 2 < p.N) yrow[n + 2] = v.z;
            }
          }
        } else {
          __nv_bfloat16* yrow = reinterpret_cast<__nv_bfloat16*>(p.Y) + (int64_t)row * p.ldy;
#pragma unroll
          for (int c = 0; c < 128; c += 8) {
            const int n = col0 + c;
            uint32_t w[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float a0 = (acc[c + 2 * h] * rs) * beta_sm[half * 128 + c + 2 * h];
              const float a1 = (acc[c + 2 * h + 1] * rs) * beta_sm[half * 128 + c + 2 * h + 1];
              const __nv_bfloat162 bb = __floats2bfloat162_rn(a0, a1);
              w[h] = *reinterpret_cast<const uint32_t*>(&bb);
            }
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
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, 512);
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

template <bool kPlain, bool kF32>
static cudaError_t launch_variant(const CUtensorMap& tx, const CUtensorMap& tw, const GemmParams& p, int grid,
                                  cudaStream_t st) {
  auto kern = rrs_gemm_kernel<kPlain, kF32>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  kern<<<grid, gemm::THREADS, gemm::SMEM_BYTES, st>>>(tx, tw, p);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmArgs& a, int nsm, cudaStream_t st) {
  using namespace gemm;
  if (a.T <= 0) return cudaSuccess;
  if (a.K / BK > MAX_G || a.K % BK) return cudaErrorInvalidValue;
  CUtensorMap tx, tw;
  if (!make_tmap(&tx, a.Xq8, a.T, a.K, BM) || !make_tmap(&tw, a.Wq8, a.N, a.K, BN)) return cudaErrorInvalidValue;
  GemmParams p;
  p.x_scale = a.x_scale;
  p.s_group = a.s_group;
  p.w_scale = a.w_scale;
  p.T = (int)a.T;
  p.N = (int)a.N;
  p.K = (int)a.K;
  p.G = (int)(a.K / BK);
  p.num_m = (int)((a.T + BM - 1) / BM);
  p.num_n = (int)((a.N + BN - 1) / BN);
  p.num_tiles = p.num_m * p.num_n;
  p.out_scale = a.out_scale;
  p.Y = a.Y;
  p.ldy = a.ldy;
  p.P_debug = a.P_debug;
  const int grid = std::min(p.num_tiles, nsm);
  const bool f32 = a.y_dtype == 1;
  if (a.plain) return f32 ? launch_variant<true, true>(tx, tw, p, grid, st) : launch_variant<true, false>(tx, tw, p, grid, st);
  return f32 ? launch_variant<false, true>(tx, tw, p, grid, st) : launch_variant<false, false>(tx, tw, p, grid, st);
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

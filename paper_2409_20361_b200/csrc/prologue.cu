// RRS runtime prologue (rows a1-a6 of SURVEY.md §8) and offline weight preparation (a7), sm_100a.
//
//   fwht_colmax_kernel : X~ = X.H (exact, fwht.cuh), c_j = max_t |X~_tj| over all T tokens
//                        (Eq. 1) via per-thread running maxima + one atomicMax per column per
//                        CTA on the float bits (valid because |x| >= +0).
//   fwht_quant_kernel  : recompute X~ (cheaper than an f32 round trip through HBM),
//                        s_g = max_{j' in g} c[perm[j']] (0 -> 1, R8), Z = X~[perm] * fl(1/s_g)
//                        (Eq. 2, R9), per-token RTN INT4 (R9-R11), pack (D4) and the
//                        int8 GEMM operand.  With chan_max == nullptr it is the weight path (a7):
//                        no smoothing (W is permuted, never scaled).
//   perm_rank_kernel   : offline reorder helper (R5): perm = argsort(c) descending, ties ascending.
#include "fwht.cuh"
#include "kernels.h"

namespace rrs {

template <int K>
__global__ void __launch_bounds__(FwhtPlan<K>::CTA)
fwht_colmax_kernel(const uint16_t* __restrict__ X, int64_t T, unsigned* __restrict__ chan_max_bits,
                   float* __restrict__ Xr_out) {
  using P = FwhtPlan<K>;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  float cm[P::SLOTS];
#pragma unroll
  for (int s = 0; s < P::SLOTS; ++s) cm[s] = 0.0f;
  for (int64_t r0 = (int64_t)blockIdx.x * P::R; r0 < T; r0 += (int64_t)gridDim.x * P::R) {
    double v[32];
    fwht_tile<P>(X, K, T, r0, sm, v);
#pragma unroll
    for (int s = 0; s < P::SLOTS; ++s) {
      int row, col;
      slot_rc<P>(tid, s, row, col);
      if (r0 + row < T) {
        const float f = __double2float_rn(v[s]);
        cm[s] = fmaxf(cm[s], fabsf(f));
        if (Xr_out) Xr_out[(r0 + row) * K + col] = f;
      }
    }
    __syncthreads();  // next tile's pass A overwrites shared memory
  }
  if ((int64_t)blockIdx.x * P::R < T) {
#pragma unroll
    for (int s = 0; s < P::SLOTS; ++s) {
      int row, col;
      slot_rc<P>(tid, s, row, col);
      atomicMax(chan_max_bits + col, __float_as_uint(cm[s]));
    }
  }
}

// max over the `width` consecutive lanes sharing a segment (width = power of two <= 32)
RRS_DEVICE float seg_max(float m, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

template <int K>
__global__ void __launch_bounds__(FwhtPlan<K>::CTA)
fwht_quant_kernel(const uint16_t* __restrict__ X, int64_t T, const int32_t* __restrict__ perm,
                  const unsigned* __restrict__ chan_max_bits, float* __restrict__ s_group_out,
                  uint8_t* __restrict__ Xq, int8_t* __restrict__ Xq8, float* __restrict__ scale_out,
                  int apply_smooth) {
  using P = FwhtPlan<K>;
  constexpr int GT = K / 32;                 // gather threads per row (32 output positions each)
  constexpr int GACT = P::R * GT;            // active gather threads
  static_assert(GACT <= P::CTA, "gather layout");
  extern __shared__ __align__(16) double sm[];
  float* fs = reinterpret_cast<float*>(sm);  // f32 X~ tile, reuses the double tile
  float* red = reinterpret_cast<float*>(sm + P::R * K);  // 64 floats of reduction scratch
  const int tid = threadIdx.x;
  const int grow = tid / GT;                 // row within tile handled in the gather phase
  const int j0 = (tid % GT) * 32;            // first reordered position j'
  const bool gact = tid < GACT;

  int pj[32];
  float inv_s = 1.0f;
  if (gact) {
    const int4* pp = reinterpret_cast<const int4*>(perm + j0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int4 w = __ldg(pp + q);
      pj[4 * q] = w.x; pj[4 * q + 1] = w.y; pj[4 * q + 2] = w.z; pj[4 * q + 3] = w.w;
    }
  }
  if (apply_smooth) {
    // s_g = max_{j' in g} c[perm[j']]  (4 consecutive threads cover one 128-wide group)
    float m = 0.0f;
    if (gact) {
#pragma unroll
      for (int k = 0; k < 32; ++k) m = fmaxf(m, __uint_as_float(__ldg(chan_max_bits + pj[k])));
    }
    m = seg_max(m, 4);
    if (m == 0.0f) m = 1.0f;  // R8: zero group -> scale 1
    inv_s = __frcp_rn(m);     // R9: fl(1/s_g)
    if (blockIdx.x == 0 && gact && grow == 0 && (j0 & 127) == 0) s_group_out[j0 >> 7] = m;
  }

  for (int64_t r0 = (int64_t)blockIdx.x * P::R; r0 < T; r0 += (int64_t)gridDim.x * P::R) {
    double v[32];
    fwht_tile<P>(X, K, T, r0, sm, v);
    __syncthreads();  // all reads of the double tile done
#pragma unroll
    for (int s = 0; s < P::SLOTS; ++s) {
      int row, col;
      slot_rc<P>(tid, s, row, col);
      fs[row * K + col] = __double2float_rn(v[s]);
    }
    __syncthreads();
    float z[32];
    float m = 0.0f;
    const int64_t trow = r0 + grow;
    if (gact) {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float x = fs[grow * K + pj[k]];
        z[k] = apply_smooth ? __fmul_rn(x, inv_s) : x;
        m = fmaxf(m, fabsf(z[k]));
      }
    }
    // per-token absmax over the GT threads of this row
    if constexpr (GT <= 32) {
      m = seg_max(m, GT);
    } else {
      m = seg_max(m, 32);
      if ((tid & 31) == 0) red[tid >> 5] = m;
      __syncthreads();
      if (gact) {
        const int w0 = (grow * GT) >> 5;
        float mm = 0.0f;
#pragma unroll 4
        for (int w = 0; w < GT / 32; ++w) mm = fmaxf(mm, red[w0 + w]);
        m = mm;
      }
    }
    if (gact && trow < T) {
      float alpha = 1.0f, r = 0.0f;
      if (m > 0.0f) {
        alpha = __fdiv_rn(m, 7.0f);  // stored scale alpha_t = fl(m/7)
        r = __fdiv_rn(7.0f, m);      // R9: codes use fl(7/m)
      }
      uint32_t packed[4] = {0u, 0u, 0u, 0u};
      uint32_t wide[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        int q = __float2int_rn(__fmul_rn(z[k], r));  // R10: round half to even
        q = max(-8, min(7, q));                      // R11
        packed[k >> 3] |= (uint32_t)(q & 0xF) << ((k & 7) * 4);
        wide[k >> 2] |= (uint32_t)(q & 0xFF) << ((k & 3) * 8);
      }
      if (Xq) {
        *reinterpret_cast<uint4*>(Xq + trow * (K / 2) + j0 / 2) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      }
      if (Xq8) {
        uint4* dst = reinterpret_cast<uint4*>(Xq8 + trow * K + j0);
        dst[0] = make_uint4(wide[0], wide[1], wide[2], wide[3]);
        dst[1] = make_uint4(wide[4], wide[5], wide[6], wide[7]);
      }
      if (j0 == 0) scale_out[trow] = alpha;
    }
    __syncthreads();  // fs / red reused by the next tile
  }
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

template <int K>
static cudaError_t launch_colmax_k(const uint16_t* X, int64_t T, unsigned* cm, float* Xr, int nsm,
                                   cudaStream_t st) {
  using P = FwhtPlan<K>;
  auto kern = fwht_colmax_kernel<K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::CTA, P::SMEM_BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = (T + P::R - 1) / P::R;
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)nsm * per_sm);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, P::CTA, P::SMEM_BYTES, st>>>(X, T, cm, Xr);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_quant_k(const uint16_t* X, int64_t T, const int32_t* perm, const unsigned* cm,
                                  float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, int nsm,
                                  cudaStream_t st) {
  using P = FwhtPlan<K>;
  auto kern = fwht_quant_kernel<K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P::CTA, P::SMEM_BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = (T + P::R - 1) / P::R;
  int grid = (int)std::min<int64_t>(tiles, (int64_t)nsm * per_sm);
  if (grid == 0) {
    if (cm == nullptr || s_group == nullptr) return cudaSuccess;
    grid = 1;  // T == 0: still publish s_group (all ones, R8)
  }
  kern<<<grid, P::CTA, P::SMEM_BYTES, st>>>(X, T, perm, cm, s_group, Xq, Xq8, scale, cm != nullptr);
  return cudaGetLastError();
}

#define RRS_FOR_EACH_K(M) M(128) M(256) M(512) M(1024) M(2048) M(4096) M(8192) M(16384) M(7168) M(14336)

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

cudaError_t launch_fwht_quant(const uint16_t* X, int64_t T, int64_t K, const int32_t* perm,
                              const unsigned* chan_max_bits, float* s_group, uint8_t* Xq, int8_t* Xq8,
                              float* scale, int nsm, cudaStream_t st) {
  switch (K) {
#define RRS_CASE(k) case k: return launch_quant_k<k>(X, T, perm, chan_max_bits, s_group, Xq, Xq8, scale, nsm, st);
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

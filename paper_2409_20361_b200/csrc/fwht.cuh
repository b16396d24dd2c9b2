// FP64-exact fast Walsh-Hadamard transform of bf16 rows for sm_100a.
//
// Computes X~ = X . H_K per row (Eq. 4; App. A.1) with the
// UNNORMALISED +-1 matrix H (R1: the 1/K = (1/sqrt K)^2 goes to the GEMM epilogue).
//   K = 2^m      : Sylvester H, butterflies over the bits of the column index.
//   K = 28 * 2^m : H28 (x) H_{2^m} (R2): FWHT-2^m on the 28 contiguous chunks, then the
//                  structured Paley-II H28 mix across chunks (S (x) A2 + I14 (x) B2, 16 adds/elem).
// Every intermediate is a signed subset sum of the row's inputs, hence exact in float64 under the
// exactness precondition (R3); the single final __double2float_rn gives the correctly
// rounded f32 value, bit-identical to the oracle's f32_rne(sum).
//
// Data movement: a CTA owns R rows at a time.  Pass A loads 32 contiguous bf16 per thread straight
// from HBM (4 x 16-byte loads) and runs 5 butterfly stages in registers; each further pass goes
// through shared memory (XOR swizzle p(i) = i ^ ((i>>5)&15) keeps every warp access at the
// 2-wavefront minimum for doubles) and runs up to 5 more stages in registers.
#pragma once
#include "common.cuh"

namespace rrs {

constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }
constexpr int max_c(int a, int b) { return a > b ? a : b; }

template <int K_>
struct FwhtPlan {
  static constexpr int K = K_;
  static constexpr bool kPow2 = (K & (K - 1)) == 0;
  static constexpr int A = kPow2 ? 1 : 28;
  static constexpr int N = K / A;             // power-of-two part
  static constexpr int LOGN = ilog2_c(N);
  static constexpr int E = 32;                // elements per thread in the 2^m passes
  static constexpr int TPR = K / E;           // threads per row in the 2^m passes
  static constexpr int H28T = kPow2 ? 0 : N;  // threads of the H28 pass (28 elements each)
  static constexpr int CTA = max_c(256, max_c(TPR, H28T));
  static constexpr int R = kPow2 ? CTA / TPR : 1;  // rows per CTA iteration
  static constexpr int SLOTS = kPow2 ? 32 : 28;    // values per thread after the last pass
  static constexpr int SMEM_BYTES = R * K * 8 + 64 * 4;  // double tile + reduction scratch
  static_assert(A * N == K, "K must be 2^m or 28*2^m");
  static_assert((N & (N - 1)) == 0 && N >= 32, "power-of-two part must be >= 32");
  static_assert(K % 128 == 0, "K must be a multiple of the group size 128");
  static_assert(CTA <= 1024, "K too large for one CTA");
  // last 2^m pass covers bits [LAST_B, LOGN)
  static constexpr int NUM_POW2_PASSES = (LOGN + 4) / 5;
  static constexpr int LAST_B = (NUM_POW2_PASSES - 1) * 5;
  static constexpr int LAST_R = LOGN - LAST_B;
};

RRS_DEVICE int swz(int i) { return i ^ ((i >> 5) & 15); }

// radix-2^r butterflies over groups v[u*2^r + k], u < 32>>r  (all stages of the pass in registers)
template <int r, int SZ>
RRS_DEVICE void butterflies(double (&v)[SZ]) {
#pragma unroll
  for (int h = 1; h < (1 << r); h <<= 1) {
#pragma unroll
    for (int u = 0; u < (SZ >> r); ++u) {
#pragma unroll
      for (int k = 0; k < (1 << r); ++k) {
        if ((k & h) == 0) {
          const double a = v[(u << r) + k], b = v[(u << r) + k + h];
          v[(u << r) + k] = a + b;
          v[(u << r) + k + h] = a - b;
        }
      }
    }
  }
}

// element index (within the R-row tile) of element k of group (tid, u) in the pass over bits [b, b+r)
template <class P, int b, int r>
RRS_DEVICE int pass_index(int tid, int u, int k) {
  const int g = tid + (P::R * P::TPR) * u;
  const int gbits = P::LOGN - r;
  const int o = g >> gbits;
  const int gx = g & ((1 << gbits) - 1);
  const int x = (gx & ((1 << b) - 1)) | (k << b) | ((gx >> b) << (b + r));
  return (o << P::LOGN) | x;
}

// Paley-II H28 = S (x) [[1,-1],[-1,-1]] + I14 (x) [[1,1],[1,-1]], S = [[0,1^T],[1,Q]], Q_ij = chi13(j-i).
// y = H28 . v  (H28 is symmetric, so row-vector x H28 == H28 x).
RRS_DEVICE int chi13(int a) {
  a = ((a % 13) + 13) % 13;
  // quadratic residues mod 13: {1, 3, 4, 9, 10, 12}
  return a == 0 ? 0 : ((a == 1 || a == 3 || a == 4 || a == 9 || a == 10 || a == 12) ? 1 : -1);
}

RRS_DEVICE void h28_apply(double (&v)[28]) {
  double u0[14], u1[14], w0[14], w1[14];
#pragma unroll
  for (int i = 0; i < 14; ++i) {
    const double x0 = v[2 * i], x1 = v[2 * i + 1];
    u0[i] = x0 - x1;      // A2 row 0: ( 1, -1)
    u1[i] = -x0 - x1;     // A2 row 1: (-1, -1)
    w0[i] = x0 + x1;      // B2 row 0: ( 1,  1)
    w1[i] = x0 - x1;      // B2 row 1: ( 1, -1)
  }
#pragma unroll
  for (int j = 0; j < 14; ++j) {
    double s0 = w0[j], s1 = w1[j];
#pragma unroll
    for (int i = 0; i < 14; ++i) {
      if (i == j) continue;
      const int sg = (j == 0 || i == 0) ? 1 : chi13((i - 1) - (j - 1));
      if (sg > 0) { s0 += u0[i]; s1 += u1[i]; } else { s0 -= u0[i]; s1 -= u1[i]; }
    }
    v[2 * j] = s0;
    v[2 * j + 1] = s1;
  }
}

// 2^m passes over bits [b, b+r), r = min(5, LOGN-b), through shared memory; the last one leaves
// its results in registers (and writes them back only if the H28 pass still has to read them).
template <class P, int b>
RRS_DEVICE void fwht_pow2_passes(double* sm, double (&v)[32]) {
  if constexpr (b < P::LOGN) {
    constexpr int r = (P::LOGN - b) < 5 ? (P::LOGN - b) : 5;
    constexpr bool last = (b + r == P::LOGN);
    const int tid = threadIdx.x;
    __syncthreads();
    if (tid < P::R * P::TPR) {
#pragma unroll
      for (int u = 0; u < (32 >> r); ++u)
#pragma unroll
        for (int k = 0; k < (1 << r); ++k) v[(u << r) + k] = sm[swz(pass_index<P, b, r>(tid, u, k))];
      butterflies<r>(v);
      if (!last || P::A == 28) {
#pragma unroll
        for (int u = 0; u < (32 >> r); ++u)
#pragma unroll
          for (int k = 0; k < (1 << r); ++k) sm[swz(pass_index<P, b, r>(tid, u, k))] = v[(u << r) + k];
      }
    }
    fwht_pow2_passes<P, b + r>(sm, v);
  }
}

// Transform rows [r0, r0+R) of X (row stride ldx elements, bf16 bits) into v[] (double).
// Rows >= T read as zero.  Ends with every thread holding SLOTS values; slot_rc() maps them.
// Contains __syncthreads(): every thread of the CTA must call it.
template <class P>
RRS_DEVICE void fwht_tile(const uint16_t* __restrict__ X, int64_t ldx, int64_t T, int64_t r0,
                          double* sm, double (&v)[32]) {
  const int tid = threadIdx.x;
  // ---- pass A: HBM -> registers, bits [0,5) ----
  if (tid < P::R * P::TPR) {
    const int rr = tid / P::TPR, tt = tid % P::TPR;
    const int64_t row = r0 + rr;
    if (row < T) {
      const uint4* src = reinterpret_cast<const uint4*>(X + row * ldx + tt * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 w = __ldg(src + q);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          v[q * 8 + 2 * h] = bf16_bits_to_double(ws[h] & 0xFFFFu);
          v[q * 8 + 2 * h + 1] = bf16_bits_to_double(ws[h] >> 16);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = 0.0;
    }
    butterflies<(P::LOGN < 5 ? P::LOGN : 5)>(v);
    if (P::NUM_POW2_PASSES > 1 || P::A == 28) {
      const int base = rr * P::K + tt * 32;
#pragma unroll
      for (int k = 0; k < 32; ++k) sm[swz(base + k)] = v[k];
    }
  }
  fwht_pow2_passes<P, 5>(sm, v);
  if constexpr (P::A == 28) {
    __syncthreads();
    // ---- H28 pass: thread x < N mixes the 28 chunk values at column offset x ----
    double w[28];
#pragma unroll
    for (int a = 0; a < 28; ++a) w[a] = sm[swz(a * P::N + tid)];
    h28_apply(w);
#pragma unroll
    for (int a = 0; a < 28; ++a) v[a] = w[a];
  }
}

// (row within tile, column) of slot s of thread tid after fwht_tile
template <class P>
RRS_DEVICE void slot_rc(int tid, int s, int& row, int& col) {
  if constexpr (P::A == 28) {
    row = 0;
    col = s * P::N + tid;
  } else if constexpr (P::NUM_POW2_PASSES == 1) {
    const int i = tid * 32 + s;
    row = i / P::K;
    col = i % P::K;
  } else {
    constexpr int b = P::LAST_B, r = P::LAST_R;
    const int i = pass_index<P, b, r>(tid, s >> r, s & ((1 << r) - 1));
    row = i / P::K;
    col = i % P::K;
  }
}

}  // namespace rrs

// FP64-exact fast Walsh-Hadamard transform of bf16 rows for sm_100a.
//
// Computes X~ = X . H_K per row (Eq. 4; App. A.1) with the
// UNNORMALISED +-1 matrix H (R1: the 1/K = (1/sqrt K)^2 goes to the GEMM epilogue).
//   K = 2^m      : Sylvester H, butterflies over the bits of the column index.
//   K = 28 * 2^m : H28 (x) H_{2^m} (R2): FWHT-2^m inside each of the 28 contiguous chunks, then
//                  the structured Paley-II H28 mix across chunks (S (x) A2 + I14 (x) B2).
// Every intermediate is a signed subset sum of the row's inputs, hence exact in float64 under the
// exactness precondition (R3); the single final __double2float_rn gives the correctly rounded
// f32 value, bit-identical to the oracle's f32_rne(sum).  The butterfly stages commute, so they may be
// run in any bit order.
//
// Data movement: every thread holds E = 2^B doubles (B = 5 for K = 2^m, 6 for 28*2^m).
// Pass 0 covers index bits {0,1,2} and the top B-3 bits of the 2^m part, so a thread's inputs are E/8 chunks
// of 8 contiguous bf16 (16-byte loads, coalesced across threads).  Each later pass covers the next (up to)
// B middle bits after one trip through shared memory; the H28 mix is one more pass.  E = 32 keeps the
// register footprint low enough for 16 warps per SM (latency hiding) at the price of a second transpose
// for K = 4096 (32 B of shared-memory traffic per element against 12 DADDs).  The padded
// address pad(i) = i + i/16 + c1*(i >> s1) + c2*(i >> s2) is strictly increasing (so injective) and, with the
// per-plan coefficients found by tools/smem_pad_search.py, gives every half-warp 16 distinct 8-byte slots
// for the pass-0 stores (stride 8), the middle passes and the H28 pass (conflict-free); it is linear in the
// register index, so every shared-memory access is one base register plus a compile-time offset.
#pragma once
#include "common.cuh"

namespace rrs {

__host__ __device__ constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }
__host__ __device__ constexpr int max_c(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int min_c(int a, int b) { return a < b ? a : b; }

// B = index bits per register pass (E = 2^B doubles per thread).  B = 5: 128 registers of values' headroom for 16 warps
// per SM, two transposes at K = 4096; B = 6 (2^m, K >= 4096): 64 doubles per thread, 8 warps per SM, one transpose
// fewer (K = 4096 = 6 + 6 bits: a single shared-memory transpose per row).
template <int K_, int B_ = 5>
struct FwhtPlan {
  static constexpr int K = K_;
  static constexpr bool kPow2 = (K & (K - 1)) == 0;
  static constexpr int A = kPow2 ? 1 : 28;          // H28 factor
  static constexpr int NP2 = K / A;                  // power-of-two part
  static constexpr int LOGN = ilog2_c(NP2);
  static constexpr int B = B_;                       // bits per pass
  static constexpr int E = 1 << B;                   // values per thread in the 2^m passes
  static constexpr int TP2 = K / E;                  // threads per row in the 2^m passes
  static constexpr int TH28 = kPow2 ? 0 : NP2;       // threads per row in the H28 pass (one 28-vector each)
  static constexpr int TPR = max_c(TP2, TH28);       // threads per row
  static constexpr int R = kPow2 ? max_c(1, (B == 5 ? 128 : 64) / TP2) : 1;  // rows per CTA tile
  static constexpr int THREADS = ((R * TPR + 31) / 32) * 32;
  static constexpr int MIN_BLOCKS = max_c(1, (B == 5 ? 512 : 256) / THREADS);  // B5: 16 warps/SM (<= 128 regs), B6: 8
  static constexpr int HI = LOGN - (B - 3);          // pass 0: bits [0,3) and [HI, LOGN)
  static constexpr int SLOTS = kPow2 ? E : 28;       // values per thread after the last pass
  static constexpr int TILE = R * K;                 // elements per CTA tile
  // padding coefficients (tools/smem_pad_search.py): B5 2^m: i + i/16 + 4(i>>7); B6 2^m (K >= 4096):
  // i + i/16 + 4(i>>8); 28*512: i + i/16; 28*256: i + i/16 + 4(i>>6) + 4(i>>8)
  static_assert(B == 5 || (kPow2 && K >= 4096), "B = 6 plans: K = 2^m >= 4096");
  static constexpr int PAD_S1 = kPow2 ? (B == 5 ? 7 : 8) : 6, PAD_C1 = (kPow2 || NP2 <= 256) ? 4 : 0;
  static constexpr int PAD_S2 = kPow2 ? 9 : 8, PAD_C2 = (!kPow2 && NP2 <= 256) ? 4 : 0;
  static constexpr int TILE_PAD = TILE + TILE / 16 + PAD_C1 * (TILE >> PAD_S1) + PAD_C2 * (TILE >> PAD_S2) + 8;
  static_assert(A * NP2 == K, "K must be 2^m or 28*2^m");
  static_assert(LOGN >= 7, "power-of-two part must be >= 128");
  static_assert(K % 128 == 0, "K must be a multiple of the group size 128");
  static_assert(THREADS <= 1024, "K too large for one CTA");
  static_assert(kPow2 || TP2 <= TH28, "H28 layout");
  static_assert(!kPow2 || E >= 32, "pow2 plan");
};

// padded shared-memory slot of tile element i (strictly increasing; max < TILE_PAD)
template <class P>
RRS_DEVICE constexpr int swz(int i) { return i + (i >> 4) + P::PAD_C1 * (i >> P::PAD_S1) + P::PAD_C2 * (i >> P::PAD_S2); }

// Input widening.  Alternative to F2F (a quarter-rate conversion on sm_100a, 16/clk/SM against 64 DADD/clk/SM:
// profiles/micro_r2.txt): the f32 bit pattern h of a bf16 value, read as the HIGH word of a double after moving its
// exponent+fraction down 3 bits (sign kept), is exactly x * 2^-896 -- the f32 and f64 exponent fields then coincide
// (e11 = e8), and f32 subnormals land on f64 subnormals with the same bits.  Every FWHT intermediate is scaled by the
// same power of two (exact: the values stay far above 2^-1074 times their f32 quantum, R3 holds unchanged), and the
// single rounding to f32 at the end first undoes the scale (one exact DMUL by 2^896).  Finite inputs only.
// Default: F2F.  The bit-move widening removes the quarter-rate conversion but costs ~4 issue slots per element
// (shift, two masks, a zeroed low word) plus the DMUL that undoes the scale, and the fused prologue is issue-bound at
// 8 warps/SM: measured A/B (bench/micro/prologue_trace vs prologue_trace_f2f, same box) 58.9 / 57.7 us with bit moves
// against 55.9 / 54.8 us with F2F at C3 up, equal at C2.  -DRRS_FWHT_BITWIDEN=1 selects the bit moves.
#ifndef RRS_FWHT_BITWIDEN
#define RRS_FWHT_BITWIDEN 0
#endif
// widen_bf16_hi: bf16 bits in the high half of h (low half zero) -> f64 (x itself, or x * 2^-896 with the bit moves);
// fwht_round_f32: an FWHT output in that representation -> the correctly rounded f32
RRS_DEVICE double widen_bf16_hi(uint32_t h) {
#if RRS_FWHT_BITWIDEN
  return __hiloint2double((int)((h & 0x80000000u) | ((h >> 3) & 0x0FFFE000u)), 0);
#else
  return (double)__uint_as_float(h);
#endif
}
RRS_DEVICE float fwht_round_f32(double d) {
#if RRS_FWHT_BITWIDEN
  return __double2float_rn(d * 0x1p896);
#else
  return __double2float_rn(d);
#endif
}

// radix-2^r butterflies over the groups v[u*2^r + k], u < E >> r (all stages of a pass in registers)
template <int r, int E>
RRS_DEVICE void butterflies(double (&v)[E]) {
#pragma unroll
  for (int h = 1; h < (1 << r); h <<= 1) {
#pragma unroll
    for (int u = 0; u < (E >> r); ++u) {
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

// Row-local index of register j = kh*8 + kl of row-thread tp in pass 0.
template <class P>
RRS_DEVICE constexpr int p0_index(int tp, int j) {
  constexpr int per_chunk = P::NP2 / P::E;  // threads per 2^m chunk
  const int a = tp / per_chunk, t = tp % per_chunk;
  return a * P::NP2 + ((j >> 3) << P::HI) + (t << 3) + (j & 7);
}

// Row-local index of element k of group u of row-thread tp in the pass over the middle bits [b, b+r).
template <class P, int b, int r>
RRS_DEVICE constexpr int p2_index(int tp, int u, int k) {
  const int g = tp + P::TP2 * u;  // the other bits, in [0, K / 2^r)
  return (g & ((1 << b) - 1)) | (k << b) | ((g >> b) << (b + r));
}

// Paley-II H28 = S (x) [[1,-1],[-1,-1]] + I14 (x) [[1,1],[1,-1]], S = [[0,1^T],[1,Q]], Q_ij = chi13(j-i).
// y = H28 . v (H28 is symmetric, so the row-vector product x H28 equals H28 x).
RRS_DEVICE constexpr int chi13(int a) {
  a = ((a % 13) + 13) % 13;
  // quadratic residues mod 13: {1, 3, 4, 9, 10, 12}
  return a == 0 ? 0 : ((a == 1 || a == 3 || a == 4 || a == 9 || a == 10 || a == 12) ? 1 : -1);
}

// y = H28 . v for the 28 values v[0..27] (pairs (x0_i, x1_i) = (v[2i], v[2i+1]), i < 14), rounded once to f32.
// With s_i = x0_i + x1_i, d_i = x0_i - x1_i the Paley-II form above gives
//   y[2j]   = s_j + (S d)_j,   y[2j+1] = d_j - (S s)_j,
//   (S u)_0 = U := sum_{i=1..13} u_i,   (S u)_j = u_0 + 2 R_j(u) - U + u_j  (j >= 1),
// where R_j(u) = sum over the 6 quadratic residues r of u_{1+((j-1+r) mod 13)}: chi13 is +1 on the residues
// and -1 on the non-residues, so sum_{i != j} chi13(i-j) u_i = 2 R_j(u) - (U - u_j).  ~10 DADD per output
// instead of ~15.  Every intermediate is a signed integer combination of the inputs no larger in magnitude
// than the final sums' bound (|2 R_j| <= 12 max|u|, |U| <= 13 max|u|), so it stays exact under R3.
RRS_DEVICE constexpr int qr13(int k) {  // the quadratic residues mod 13
  return k == 0 ? 1 : k == 1 ? 3 : k == 2 ? 4 : k == 3 ? 9 : k == 4 ? 10 : 12;
}
template <int E, class Emit>
RRS_DEVICE void h28_lean(double (&v)[E], Emit&& emit) {
#pragma unroll
  for (int i = 0; i < 14; ++i) {
    const double a = v[2 * i], b = v[2 * i + 1];
    v[2 * i] = a + b;      // s_i
    v[2 * i + 1] = a - b;  // d_i
  }
  double S = 0.0, D = 0.0;
#pragma unroll
  for (int i = 1; i < 14; ++i) {
    S += v[2 * i];
    D += v[2 * i + 1];
  }
  emit(0, fwht_round_f32(v[0] + D));
  emit(1, fwht_round_f32(v[1] - S));
#pragma unroll
  for (int j = 1; j < 14; ++j) {
    double rs = 0.0, rd = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int i = 1 + ((j - 1 + qr13(k)) % 13);
      rs += v[2 * i];
      rd += v[2 * i + 1];
    }
    const double sj = v[2 * j], dj = v[2 * j + 1];
    emit(2 * j, fwht_round_f32(fma(2.0, rd, (sj + dj) + (v[1] - D))));
    emit(2 * j + 1, fwht_round_f32(dj - fma(2.0, rs, (sj + v[0]) - S)));
  }
}

// ------------------------------------------------------------------------------ pass plumbing
// A "layout" names which index each register holds: pass 0 (L = -1), a middle pass starting at bit b
// (L = b), or the H28 pass (L = -2).

template <class P, int L>
RRS_DEVICE constexpr int reg_index(int tp, int j) {
  if constexpr (L == -1) {
    return p0_index<P>(tp, j);
  } else if constexpr (L == -2) {
    // register j = chunk index; the thread's column offset inside the 2^m chunk is tp
    return j * P::NP2 + tp;
  } else {
    constexpr int r = min_c(P::B, P::HI - L);
    return p2_index<P, L, r>(tp, j >> r, j & ((1 << r) - 1));
  }
}

// In the pass-0 and H28 layouts of every plan, and in every layout of the 2^m plans, the tile index splits into disjoint
// bit fields: the row and thread part reg_index(tp, 0) and the register part reg_index(0, j)
// (tests/test_fwht_layout_cpu.py).  Disjoint fields add without carries, so every shift in swz distributes over them:
// swz(rr K + reg_index(tp, j)) = swz(rr K + reg_index(tp, 0)) + swz(reg_index(0, j)) -- one base address per pass and a
// compile-time offset per register.  (The middle passes of 28 * 2^m plans, whose thread count 16 * 28 is not a power of
// two, compute each address.)
template <class P, int L>
__host__ __device__ constexpr bool separable() { return P::kPow2 || L < 0; }

template <class P, int L>
RRS_DEVICE void store_layout(double* sm, int rr, int tp, const double (&v)[P::E]) {
  constexpr int n = (L == -2) ? 28 : P::E;
  if constexpr (separable<P, L>()) {
    double* base = sm + swz<P>(rr * P::K + reg_index<P, L>(tp, 0));
#pragma unroll
    for (int j = 0; j < n; ++j) base[swz<P>(reg_index<P, L>(0, j))] = v[j];
  } else {
#pragma unroll
    for (int j = 0; j < n; ++j) sm[swz<P>(rr * P::K + reg_index<P, L>(tp, j))] = v[j];
  }
}

template <class P, int L>
RRS_DEVICE void load_layout(const double* sm, int rr, int tp, double (&v)[P::E]) {
  constexpr int n = (L == -2) ? 28 : P::E;
  if constexpr (separable<P, L>()) {
    const double* base = sm + swz<P>(rr * P::K + reg_index<P, L>(tp, 0));
#pragma unroll
    for (int j = 0; j < n; ++j) v[j] = base[swz<P>(reg_index<P, L>(0, j))];
  } else {
#pragma unroll
    for (int j = 0; j < n; ++j) v[j] = sm[swz<P>(rr * P::K + reg_index<P, L>(tp, j))];
  }
}

// The middle passes [b, HI) following a pass with layout PL; finally the H28 pass.  Ends with v in the
// layout last_layout<P>().  Every thread of the CTA must call it.  `staged()` runs (in every thread) right after the
// first CTA barrier, when every thread has consumed its pass-0 inputs (the bf16 stage may be refilled).
template <class P, int PL, int b, class Emit, class Hook>
RRS_DEVICE void fwht_rest(double* sm, int rr, int tp, bool p2act, bool h28act, double (&v)[P::E], Emit&& emit,
                          Hook&& staged) {
  if constexpr (b < P::HI) {
    constexpr int r = min_c(P::B, P::HI - b);
    if (p2act) store_layout<P, PL>(sm, rr, tp, v);
    __syncthreads();
    if constexpr (PL == -1) staged();
    if (p2act) {
      load_layout<P, b>(sm, rr, tp, v);
      butterflies<r>(v);
    }
    __syncthreads();  // the tile is rewritten by the next pass (or by the next row)
    fwht_rest<P, b, b + r>(sm, rr, tp, p2act, h28act, v, emit, staged);
  } else if constexpr (!P::kPow2) {
    if (p2act) store_layout<P, PL>(sm, rr, tp, v);
    __syncthreads();
    if constexpr (PL == -1) staged();
    if (h28act) {
      load_layout<P, -2>(sm, 0, threadIdx.x, v);  // H28 layout is indexed by the CTA thread
      h28_lean(v, emit);
    }
    __syncthreads();
  }
}

template <class P>
__host__ __device__ constexpr int last_layout() {
  if constexpr (!P::kPow2) return -2;
  int b = 3, last = -1;
  while (b < P::HI) {
    last = b;
    b += min_c(P::B, P::HI - b);
  }
  return last;
}

// Transform the R-row bf16 tile `stage` (shared memory, raw bits, row-major [R][K]); v[] is scratch.
// For every j < SLOTS of an active thread (out_active), calls emit(j, y) with y the correctly rounded (f32)
// rotated value of row-local column out_col<P>(tp, j) of tile row rr (t = rr * TP2 + tp in the 2^m passes;
// t = tp for H28).  rr and tp are set before the first emit.
// active_rows masks rows beyond the matrix (their lanes still run, on whatever the stage holds).
// (tile row, row-thread) of CTA thread t in the last layout: the rr / tp that fwht_tile passes to its emits
template <class P>
RRS_DEVICE void tile_coords(int t, int& rr, int& tp) {
  const bool p2act = t < P::R * P::TP2;
  rr = P::kPow2 ? (p2act ? t / P::TP2 : 0) : 0;
  tp = P::kPow2 ? (p2act ? t % P::TP2 : 0) : t;
}

template <class P, class Emit, class Hook>
RRS_DEVICE void fwht_tile(const uint16_t* stage, double* sm, double (&v)[P::E], int& rr, int& tp, Emit&& emit,
                          Hook&& staged) {
  const int t = threadIdx.x;
  const bool p2act = t < P::R * P::TP2;
  const bool h28act = !P::kPow2 && t < P::TH28;
  rr = P::kPow2 ? (p2act ? t / P::TP2 : 0) : 0;
  const int tp2 = p2act ? t % P::TP2 : 0;
  tp = P::kPow2 ? tp2 : t;
  if (p2act) {
    // bf16 -> f64 (exact for every finite value incl. subnormals; widen_bf16_hi)
    const uint16_t* row = stage + rr * P::K;
#pragma unroll
    for (int kh = 0; kh < P::E / 8; ++kh) {
      const uint4 w = *reinterpret_cast<const uint4*>(row + p0_index<P>(tp2, kh * 8));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[kh * 8 + 2 * h] = widen_bf16_hi(ws[h] << 16);
        v[kh * 8 + 2 * h + 1] = widen_bf16_hi(ws[h] & 0xFFFF0000u);
      }
    }
    butterflies<P::B>(v);
  }
  fwht_rest<P, -1, 3>(sm, rr, tp2, p2act, h28act, v, emit, staged);
  if constexpr (P::kPow2) {
    if (p2act) {
#pragma unroll
      for (int j = 0; j < P::SLOTS; ++j) emit(j, fwht_round_f32(v[j]));
    }
  }
}
template <class P, class Emit>
RRS_DEVICE void fwht_tile(const uint16_t* stage, double* sm, double (&v)[P::E], int& rr, int& tp, Emit&& emit) {
  fwht_tile<P>(stage, sm, v, rr, tp, emit, [] {});
}

template <class P>
RRS_DEVICE constexpr int out_col(int tp, int j) {
  return reg_index<P, last_layout<P>()>(tp, j);
}

template <class P>
RRS_DEVICE bool out_active(int t) {
  return P::kPow2 ? t < P::R * P::TP2 : t < P::TH28;
}

}  // namespace rrs

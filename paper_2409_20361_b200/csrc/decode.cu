// Decode-regime RRS GEMM (BASELINE configs[3]: 1-64 tokens x K = 8192 x N = 8192), sm_100a.
//
// Same arithmetic as rrs_gemm_kernel (fig:framework (3) P:103):
//   P_g[t][n] = sum_{j' in g} q[t][j'] qw[n][j']   (exact int32 in TMEM)
//   Y[t][n]   = (sum_g s_g P_g[t][n]) * (alpha_t * out_scale) * beta_n
// but built for a W stream: at T <= 64 the layer is bound by reading W from HBM (N K codes), so W stays PACKED
// at 4 bits in HBM (half the bytes of the one-code-per-byte prefill operand) and is widened on chip.
//
//   * swap-AB: the MMA's M = 128 lanes are W rows (A operand), its N = the T tokens padded to TP (B operand);
//   * A is read from TENSOR MEMORY: converter warps widen the packed nibbles to int8 in registers and
//     tcgen05.st them into a TMEM stage, so the widened W never touches shared memory (the SMEM path would be
//     shared-memory-bandwidth bound: TMA write + widen read + widened write + MMA read per code);
//   * packed layout ("decode4", produced offline by rrs_prepare_weights(RRS_W_PACKED4)): per row, per 32-code
//     chunk j0..j0+31, byte b (0..15) = (q[j0+b] << 4) | (q[j0+16+b] & 0xF).  Widening is then two masks per
//     32-bit word: (w & 0xF0F0F0F0) holds 16 q[j0+4i..] as int8 bytes, ((w << 4) & 0xF0F0F0F0) holds 16 q[j0+16+4i..],
//     i.e. the MMA sums 16 P_g exactly (|16 P_g| <= 16 * 6272 < 2^17) and the promotion scale is s_g / 16;
//   * each CTA owns 256 W rows (two M = 128 halves sharing every X tile) and a contiguous range of K-blocks;
//     the S CTAs that split a row block's K form a cluster and reduce their f32 partials through DSMEM in a
//     fixed rank order (deterministic, R15) -- no global scratch, no memset, no second kernel;
//   * the W ring starts filling BEFORE griddepcontrol.wait (W does not depend on the prologue), so with
//     programmatic dependent launch the W stream overlaps the prologue's tail.
// Warps: 0 TMA producer, 1 TMEM allocator + single-thread MMA issuer, 2-5 converters (W nibbles -> TMEM),
// 6-13 promotion (TMEM P_g -> registers, acc += s_g P_g) + epilogue.
#include <algorithm>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "kernels.h"
#include "ptx.cuh"

namespace rrs {

// Optional timeline (tools/decode_trace.cu builds this file with -DRRS_TRACE): %globaltimer per CTA (< 8), per
// event (W issued, X issued, converted, MMA issued, promoted, start, end) and K-block (< 64).
#ifdef RRS_TRACE
__device__ unsigned long long g_dtrace[8][8][64];
__device__ __forceinline__ void dtrace(int ev, int i) {
  if (blockIdx.x < 8 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dtrace[blockIdx.x][ev][i] = t;
  }
}
// experiment knobs of the timeline harness: bit 0 = load X only for the first ring round (W-stream-only timing)
__device__ int g_dec_exp = 0;
int g_dec_no_pdl = 0;  // host: launch the GEMM without programmatic dependent launch
#else
__device__ __forceinline__ void dtrace(int, int) {}
#endif

namespace dec {
constexpr int ROWS = 256;                // W rows per CTA (two MMA halves of 128)
constexpr int KBLK = 128;                // codes per K-block
constexpr int W_STAGE = ROWS * KBLK / 2; // packed W bytes per K-block: one contiguous 16 KiB tile
constexpr int NS = 8;                    // W ring stages
constexpr int min_i(int a, int b) { return a < b ? a : b; }
constexpr int NA = 3;                    // TMEM A stages (widened W)
constexpr int NCONV = 4, NPROM = 8;
constexpr int W_PROD = 0, MMA_WARP = 1, CONV0 = 2, PROM0 = CONV0 + NCONV, X_PROD = PROM0 + NPROM;
constexpr int THREADS = (X_PROD + 1) * 32;
constexpr int A_COL0 = 256;              // TMEM columns [256, 256 + 64 NA): A stages; [0, 4 TP): accumulators
constexpr int MAX_G = 160;

template <int TP>
struct Cfg {
  static constexpr int X_STAGE = TP * KBLK;   // int8 X codes per K-block (SWIZZLE_128B tile)
  static constexpr int NX = min_i(16, 65536 / X_STAGE);  // X ring: 8 stages at TP = 64, 16 below (X loads are L2 hits
                                                         // whose latency must not sit in the per-K-block loop)
  static constexpr int X_OFF = NS * W_STAGE;
  static constexpr int RING = X_OFF + NX * X_STAGE;
  static constexpr int ROWB = (TP + 4) * 4;      // one row of partials (f32, 16-byte aligned stride)
  // after the K loop, on the ring: this CTA's partials [256][TP + 4] f32, then the S incoming slots
  // [S][256/S][TP + 4] (the same 256 rows' worth of bytes)
  static constexpr int RED = 2 * ROWS * ROWB;
  static constexpr int SMEM = 1024 + RING + 1024 + MAX_G * 4 + 64 * 4 + ROWS * 4;  // + s_g, alpha_t, beta_n
  static_assert(X_STAGE % 1024 == 0 && W_STAGE % 1024 == 0, "1024-byte aligned swizzle atoms");
  static_assert(RED <= RING, "reduction overlay");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};
}  // namespace dec

struct DecodeParams {
  const uint8_t* Wp4;  // tiled decode4 layout [ceil(N/256)][K/128][16 KiB]
  const float* x_scale;
  const float* s_group;
  const float* w_scale;
  int T, N, K;
  int kb_per_cta;   // K-blocks per CTA (a whole number of groups)
  int gpb;          // K-blocks per smoothing group
  int S;            // CTAs per cluster (split-K)
  float out_scale;
  void* Y;
  int y_f32;
  int64_t ldy;
};

template <int TP>
__global__ void __launch_bounds__(dec::THREADS, 1)
rrs_decode_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x, DecodeParams p) {
  using namespace dec;
  using C = Cfg<TP>;
  constexpr int NX = C::NX;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* wring = smem;                                  // [NS][16 KiB] packed W tiles
  uint8_t* xring = smem + C::X_OFF;                       // [NX][TP x 128] int8 X codes
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::RING);
  uint64_t* wfull = bars;
  uint64_t* wempty = wfull + NS;
  uint64_t* xfull = wempty + NS;
  uint64_t* xempty = xfull + NX;
  uint64_t* afull = xempty + NX;
  uint64_t* aempty = afull + NA;
  uint64_t* tfull = aempty + NA;
  uint64_t* tempty = tfull + 2;
  uint64_t* redbar = tempty + 2;     // the peers' partial slices have landed (bulk copies, complete_tx)
  uint32_t* taddr_slot = reinterpret_cast<uint32_t*>(redbar + 1);
  float* s_sm = reinterpret_cast<float*>(smem + C::RING + 1024);
  float* xs_sm = s_sm + MAX_G;   // alpha_t * out_scale, t < T
  float* ws_sm = xs_sm + 64;     // beta_n of this CTA's 256 rows (0 past N)
  float* part = reinterpret_cast<float*>(wring);          // after the K loop: own partials [256][TP + 4]
  float* slots = part + ROWS * (TP + 4);                   // incoming [S][256/S][TP + 4]

  const uint32_t warp = ptx::warp_idx();
  const int lane = threadIdx.x & 31;
  const int S = p.S;
  const uint32_t rank = S > 1 ? ptx::cluster_ctarank() : 0u;
  const int rb = blockIdx.x / S;
  const int row0 = rb * ROWS;
  const int nkb = p.kb_per_cta;
  const int kb0 = (int)rank * nkb;
  const int ng = nkb / p.gpb;
  const int g0 = kb0 / p.gpb;
  const int rows_per = ROWS / S;
  // every row block walks its K range starting at a different group (rotated by the row block): the X tiles are shared
  // by all row blocks, and CTAs requesting the same X tile at the same moment serialise on its L2 lines.  The group
  // order of the promotion differs per row block but is fixed (R15).
  const int rot = rb % ng;
  auto kb_at = [&](int i) { return ((i / p.gpb + rot) % ng) * p.gpb + i % p.gpb; };  // loop index -> K-block (CTA range)

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], NCONV);
    }
    for (int s = 0; s < NX; ++s) {
      ptx::mbar_init(&xfull[s], 1);
      ptx::mbar_init(&xempty[s], 1);
    }
    for (int a = 0; a < NA; ++a) {
      ptx::mbar_init(&afull[a], NCONV);
      ptx::mbar_init(&aempty[a], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], NPROM);
    }
    ptx::mbar_init(redbar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x == 0) dtrace(5, 0);
  if (warp == MMA_WARP) ptx::tmem_alloc(taddr_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *taddr_slot;

  if (warp == W_PROD) {
    // ------------------------------------------------------------------ W stream: one 16 KiB bulk copy per K-block
    // (W does not depend on the prologue: no griddepcontrol.wait, the ring fills while the prologue finishes)
    if (ptx::elect_one()) {
      const uint8_t* wsrc = p.Wp4 + ((int64_t)rb * (p.K / KBLK) + kb0) * W_STAGE;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % NS;
        ptx::mbar_wait(&wempty[s], ((i / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&wfull[s], W_STAGE);
        ptx::bulk_load(wring + s * W_STAGE, wsrc + (int64_t)kb_at(i) * W_STAGE, W_STAGE, &wfull[s]);
        dtrace(0, i);
      }
    }
  } else if (warp == X_PROD) {
    // ------------------------------------------------------------------ X codes (from the prologue), own ring
    if (ptx::elect_one()) {
      ptx::pdl_wait();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % NX;
        ptx::mbar_wait(&xempty[s], ((i / NX) & 1) ^ 1);
#ifdef RRS_TRACE
        if ((g_dec_exp & 1) && i >= NX) {
          ptx::mbar_arrive_expect_tx(&xfull[s], 0);
          continue;
        }
#endif
        ptx::mbar_arrive_expect_tx(&xfull[s], C::X_STAGE);
        ptx::tma_load_2d(xring + s * C::X_STAGE, &tmap_x, &xfull[s], (kb0 + kb_at(i)) * KBLK, 0, ptx::kEvictLast);
        dtrace(1, i);
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_i8(128, TP);
      const uint64_t xdesc0 = ptx::smem_desc_sw128(xring);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % NX, a = i % NA;
        const int gl = i / p.gpb, kin = i % p.gpb;
        const uint32_t b = gl & 1;
        if (kin == 0) ptx::mbar_wait(&tempty[b], ((gl >> 1) & 1) ^ 1);
        ptx::mbar_wait(&afull[a], (i / NA) & 1);
        ptx::mbar_wait(&xfull[s], (i / NX) & 1);
        ptx::tc_fence_after();
        const uint64_t xdesc = xdesc0 + (uint64_t)((s * C::X_STAGE) >> 4);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int k = 0; k < KBLK / 32; ++k)
            ptx::mma_i8_ts(tmem + b * (2 * TP) + h * TP, tmem + A_COL0 + a * 64 + h * 32 + k * 8, xdesc + 2 * k, idesc,
                           (kin > 0 || k > 0) ? 1u : 0u);
        ptx::mma_commit(&aempty[a]);
        ptx::mma_commit(&xempty[s]);
        if (kin == p.gpb - 1) ptx::mma_commit(&tfull[b]);
        dtrace(3, i);
      }
    }
    __syncwarp();
  } else if (warp < PROM0) {
    // ------------------------------------------------------------------ converters: packed W -> int8 in TMEM
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % NS, a = i % NA;
      ptx::mbar_wait(&wfull[s], (i / NS) & 1);
      ptx::mbar_wait(&aempty[a], ((i / NA) & 1) ^ 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = h * 128 + q * 32 + lane;
        // the tile is stored pre-swizzled: 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3), so every
        // quarter-warp's 16-byte loads hit 8 distinct bank groups
        const uint8_t* rowp = wring + s * W_STAGE + r * 64;
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 w = *reinterpret_cast<const uint4*>(rowp + ((c ^ ((r >> 1) & 3)) << 4));
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            v[8 * c + j] = ww[j] & 0xF0F0F0F0u;             // 16 q[j0 + 4j ..]     (high nibbles)
            v[8 * c + 4 + j] = (ww[j] << 4) & 0xF0F0F0F0u;  // 16 q[j0 + 16 + 4j ..] (low nibbles)
          }
        }
        RRS_TMEM_ST32(tmem + lane_off + A_COL0 + a * 64 + h * 32, v);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&wempty[s]);
        ptx::mbar_arrive(&afull[a]);
        if (warp == CONV0) dtrace(2, i);
      }
    }
  } else {
    // ------------------------------------------------------------------ promotion
    const int q = warp & 3, h = (warp - PROM0) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    ptx::pdl_wait();  // s_g come from the prologue
    for (int g = threadIdx.x - PROM0 * 32; g < ng; g += NPROM * 32) s_sm[g] = p.s_group[g0 + g];
    {  // the epilogue's scales, read once here (off the critical path)
      const int i = threadIdx.x - PROM0 * 32;  // 0 .. 255
      if (i < p.T) xs_sm[i] = p.x_scale[i] * p.out_scale;
      ws_sm[i] = row0 + i < p.N ? p.w_scale[row0 + i] : 0.0f;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NPROM * 32));
    float acc[TP];  // sum_g s_g P_g of this thread's W row for the TP token columns
#pragma unroll
    for (int t = 0; t < TP; ++t) acc[t] = 0.0f;
    for (int gl = 0; gl < ng; ++gl) {
      const uint32_t b = gl & 1;
      ptx::mbar_wait(&tfull[b], (gl >> 1) & 1);
      ptx::tc_fence_after();
      if (warp == PROM0 && lane == 0) dtrace(4, gl);
      const float sc = s_sm[(gl + rot) % ng] * 0.0625f;  // s_g / 16 (exact: the widened codes are 16 q)
      // the group's loads two at a time, one wait per pair (the load latency, not its bandwidth, paced the MMA)
#pragma unroll
      for (int c = 0; c < TP / 16; c += 2) {
        uint32_t v[32];
        RRS_TMEM_LD16(tmem + lane_off + b * (2 * TP) + h * TP + c * 16, v);
        if (c + 1 < TP / 16) RRS_TMEM_LD16(tmem + lane_off + b * (2 * TP) + h * TP + (c + 1) * 16, (v + 16));
        RRS_TMEM_WAIT_LD16(v);
        if (c + 1 < TP / 16) RRS_REG_FENCE16((v + 16));
        if (c + 2 >= TP / 16) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[b]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 16 + j < TP) acc[c * 16 + j] = fmaf(sc, (float)(int)v[j], acc[c * 16 + j]);
      }
    }
    // every MMA has completed (this warp saw the last tfull), so every converter and every ring stage of this CTA
    // is done (the CTA barrier below states it directly as well); the partials then go to this CTA's own ring
    // (16-byte stores, row stride TP + 4 floats) and a proxy fence makes them visible to the bulk copies
    if (warp == PROM0 && lane == 0) dtrace(7, 0);
    asm volatile("barrier.sync 2, %0;" ::"n"(THREADS) : "memory");
    const int r = h * 128 + q * 32 + lane;
#pragma unroll
    for (int t4 = 0; t4 < TP / 4; ++t4)
      if (4 * t4 < p.T)
        *reinterpret_cast<float4*>(part + r * (TP + 4) + 4 * t4) =
            make_float4(acc[4 * t4], acc[4 * t4 + 1], acc[4 * t4 + 2], acc[4 * t4 + 3]);
    ptx::fence_proxy_async_shared();
  }
  // the other warps' arrival at that CTA barrier (non-aligned form: producer lanes may still be diverged)
  if (warp < PROM0 || warp >= PROM0 + NPROM) asm volatile("barrier.sync 2, %0;" ::"n"(THREADS) : "memory");
  // first cluster barrier: every CTA of the cluster is done with its ring (the peers' slots are free) and has its
  // partials in place
  ptx::tc_fence_before();
  if (S > 1) ptx::cluster_sync();
  else __syncthreads();
  if (warp == PROM0 && lane == 0) dtrace(7, 1);
  // the owner of rows [r 256/S, (r+1) 256/S) is rank r: one bulk copy (TMA) per peer of that contiguous slice into the
  // peer's slot [my rank], completing on the peer's redbar -- shared-memory-to-shared-memory over the cluster
  const uint32_t slice_bytes = (uint32_t)(rows_per * (TP + 4) * 4);
  if (threadIdx.x == 0 && S > 1) {
    ptx::mbar_arrive_expect_tx(redbar, (uint32_t)(S - 1) * slice_bytes);
    for (int o = 0; o < S; ++o) {
      if (o == (int)rank) continue;
      ptx::bulk_copy_cta_to_peer(slots + ((int)rank * rows_per) * (TP + 4), (uint32_t)o,
                                 part + (o * rows_per) * (TP + 4), slice_bytes, redbar);
    }
  }
  if (S > 1) {
    ptx::mbar_wait(redbar, 0);  // the S - 1 incoming slices have landed
    ptx::cluster_sync_warps_arrive();  // ... so every copy out of a peer's partials has completed (joined at the end)
  }
  __syncthreads();  // (already implied by the cluster barrier above; stated for the shared-memory race checker)
  if (threadIdx.x == 0) dtrace(7, 2);
  // ---- fixed-order reduction over the S slots (ranks 0..S-1) and the epilogue: rank r writes rows
  // [r 256/S, (r+1) 256/S) of the row block
  {
    const int nout = ((p.T + 3) / 4) * rows_per;  // (4 tokens, 1 row) per item
    for (int idx = threadIdx.x; idx < nout; idx += THREADS) {
      const int tg = idx / rows_per, rr = idx % rows_per;
      const int n = row0 + (int)rank * rows_per + rr;
      float4 sum = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      for (int src = 0; src < S; ++src) {  // fixed rank order (R15); this CTA's own slice straight from part
        const float* row = src == (int)rank ? part + ((int)rank * rows_per + rr) * (TP + 4)
                                            : slots + (src * rows_per + rr) * (TP + 4);
        const float4 v = *reinterpret_cast<const float4*>(row + 4 * tg);
        sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
      }
      if (n < p.N) {
        const float bn = ws_sm[(int)rank * rows_per + rr];
        const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int t = 4 * tg + i;
          if (t < p.T) {
            const float y = sv[i] * xs_sm[t] * bn;
            if (p.y_f32) reinterpret_cast<float*>(p.Y)[(int64_t)t * p.ldy + n] = y;
            else reinterpret_cast<__nv_bfloat16*>(p.Y)[(int64_t)t * p.ldy + n] = __float2bfloat16_rn(y);
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) dtrace(6, 0);
  if (S > 1) ptx::cluster_wait();  // no CTA exits while a peer's bulk copy may still read its partials
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == MMA_WARP) ptx::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn_dec() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t row_bytes, int box_bytes, int box_rows,
                     CUtensorMapSwizzle sw) {
  auto fn = encode_fn_dec();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_bytes, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TP>
static cudaError_t launch_decode_tp(const CUtensorMap& tx, const DecodeParams& p, int grid, cudaStream_t st) {
  auto kern = rrs_decode_gemm_kernel<TP>;
  constexpr int smem = dec::Cfg<TP>::SMEM;
  cudaError_t e = prepare_kernel(kern, smem, dec::THREADS);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dec::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
#ifdef RRS_TRACE
  if (g_dec_no_pdl) cfg.numAttrs = 1;  // timeline experiment: the GEMM starts only after the prologue has finished
#endif
  return cudaLaunchKernelEx(&cfg, kern, tx, p);
}

bool decode_gemm_supports(int64_t T, int64_t K, int group) {
  return T >= 1 && T <= 64 && group >= 128 && group % 128 == 0 && K % group == 0 && K / group <= dec::MAX_G;
}

cudaError_t launch_decode_gemm(const DecodeArgs& a, int nsm, cudaStream_t st) {
  using namespace dec;
  if (a.T <= 0) return cudaSuccess;
  if (!decode_gemm_supports(a.T, a.K, a.group)) return cudaErrorInvalidValue;
  const int KBt = (int)(a.K / KBLK), G = (int)(a.K / a.group), gpb = a.group / KBLK;
  const int R = (int)((a.N + ROWS - 1) / ROWS);
  // split K over a cluster of S CTAs (whole groups each) while the grid still fits on the SMs
  int S = 1;
  for (int s : {2, 4, 8})
    if (G % s == 0 && (int64_t)R * s <= nsm) S = s;
  CUtensorMap tx;
  const int TP = a.T <= 16 ? 16 : a.T <= 32 ? 32 : 64;
  if (!make_map(&tx, a.Xq8, a.T, a.K, 128, TP, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  DecodeParams p;
  p.Wp4 = a.Wp4;
  p.x_scale = a.x_scale;
  p.s_group = a.s_group;
  p.w_scale = a.w_scale;
  p.T = (int)a.T;
  p.N = (int)a.N;
  p.K = (int)a.K;
  p.kb_per_cta = KBt / S;
  p.gpb = gpb;
  p.S = S;
  p.out_scale = a.out_scale;
  p.Y = a.Y;
  p.y_f32 = a.y_dtype == 1;
  p.ldy = a.ldy;
  const int grid = R * S;
  if (TP == 16) return launch_decode_tp<16>(tx, p, grid, st);
  if (TP == 32) return launch_decode_tp<32>(tx, p, grid, st);
  return launch_decode_tp<64>(tx, p, grid, st);
}

}  // namespace rrs

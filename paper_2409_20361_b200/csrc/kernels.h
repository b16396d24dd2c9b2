// Internal host-side launch entry points of the RRS kernels (not part of the public C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rrs {

// Per-(kernel, device) one-time setup: the dynamic shared-memory opt-in and the occupancy query are host
// calls that cost microseconds; do them once per kernel function and device, not on every launch.
struct KernelPrep {
  const void* fn;
  int dev, per_sm;
};
cudaError_t prepare_kernel_impl(const void* fn, int smem, int threads, int* blocks_per_sm);
template <class F>
cudaError_t prepare_kernel(F kern, int smem, int threads, int* blocks_per_sm = nullptr) {
  return prepare_kernel_impl(reinterpret_cast<const void*>(kern), smem, threads, blocks_per_sm);
}

// Per-(kernel, device) cached cudaOccupancyMaxActiveClusters for a kernel with compile-time cluster dims
// (0 if the query fails).  Thread-safe.
int max_active_clusters_impl(const void* fn, int cluster, int threads, int smem);
template <class F>
int max_active_clusters(F kern, int cluster, int threads, int smem) {
  return max_active_clusters_impl(reinterpret_cast<const void*>(kern), cluster, threads, smem);
}

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int threads, int smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}


bool prologue_supports_k(int64_t K);
cudaError_t launch_fwht_colmax(const uint16_t* X, int64_t T, int64_t K, unsigned* chan_max_bits, float* Xr,
                               int nsm, cudaStream_t st);
// One persistent (cooperative) launch of rows a1-a6 for K = 2^m that reduces group maxima only (no chan_max output;
// no zeroed input).  Returns cudaErrorCooperativeLaunchTooLarge when the grid cannot be co-resident.
bool prologue_fused_supports_k(int64_t K);
cudaError_t launch_prologue_fused(const uint16_t* X, int64_t T, int64_t K, float* Xr, const int32_t* perm,
                                  float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3, int group,
                                  cudaStream_t st);
// Decode-sized T (1..64, K = 2^m in [1024, 8192]): rows a1-a6 in one cooperative launch, one CTA per row, the FWHT
// of a row spread over its K/1024 warps; no memset (chan_max is written, not accumulated).  scratch: >= T * K f32.
bool prologue_decode_supports(int64_t T, int64_t K, int group);
cudaError_t launch_prologue_decode(const uint16_t* X, int64_t T, int64_t K, const int32_t* perm, unsigned* chan_max_bits,
                                   float* scratch, float* s_group, uint8_t* Xq, int8_t* Xq8, float* scale, bool e4m3,
                                   int group, cudaStream_t st);
// X~ = X (bf16 -> f32, no rotation) and, unless chan_max_bits is null, the runtime channel max (atomicMax on
// zeroed float bits) -- the RRS_NO_ROTATION / RRS_PREROTATED prologue and the NO_ROTATION weight path
cudaError_t launch_convert_colmax(const uint16_t* X, int64_t T, int64_t K, unsigned* chan_max_bits, float* Xr, int nsm,
                                  cudaStream_t st);
// chan_max_bits == nullptr: weight mode (no smoothing, s_group unused).  dec4: Xq in the decode4 nibble layout
// (rrs.h RRS_W_PACKED4) instead of D4.
cudaError_t launch_smooth_quant(const float* Xr, int64_t T, int64_t K, const int32_t* perm,
                                const unsigned* chan_max_bits, float* s_group, uint8_t* Xq, int8_t* Xq8,
                                float* scale, bool e4m3, int group, int nsm, cudaStream_t st, bool dec4 = false);
cudaError_t launch_perm_rank(const float* c, int64_t K, int32_t* perm, cudaStream_t st);

struct GemmArgs {
  const int8_t* Xq8;      // [T][K] int8 codes (reordered order)
  const float* x_scale;   // [T]
  const float* s_group;   // [G]
  const int8_t* Wq8;      // [N][K]
  const float* w_scale;   // [N]
  int64_t T, N, K;
  int group;
  float out_scale;
  bool plain;             // per-channel A4W4 baseline: one accumulation over all K, no s_g
  bool fp8;               // operand codes are E4M3 bytes (kind::f8f6f4, exact FP32 sums) instead of int8
  void* Y;                // [T][ldy]
  int y_dtype;            // 0 = bf16, 1 = f32
  int64_t ldy;
  int32_t* P_debug;       // optional [G][T][N] export of the int32 group partials (test only)
  bool swiglu = false;    // bf16 Y[T][N/2] = silu(gate) * up of interleaved (gate_i, up_i) rows
  int splits = 1;         // split-K: >1 writes f32 partials [splits][T][ldy] to Y (then launch_reduce_splits)
  bool subchannel = false; // SURVEY §8 f4 baseline: x_scale alpha[G][T], w_scale beta[G][N], no s_group
};
// Y = sum of the split-K partials [splits][T][N] f32 (fixed order), f32 or bf16 out
cudaError_t launch_reduce_splits(const float* part, int splits, int64_t T, int64_t N, void* Y, int y_dtype,
                                 int64_t ldy, cudaStream_t st);
cudaError_t launch_gemm(const GemmArgs& a, int nsm, cudaStream_t st);

// Decode-regime GEMM (decode.cu): int8 X codes [T][K] x decode4-packed W [N][K/2], T <= 64, group % 128 == 0
struct DecodeArgs {
  const int8_t* Xq8;
  const float* x_scale;
  const float* s_group;
  const uint8_t* Wp4;
  const float* w_scale;
  int64_t T, N, K;
  int group;
  float out_scale;
  void* Y;
  int y_dtype;  // 0 = bf16, 1 = f32
  int64_t ldy;
};
bool decode_gemm_supports(int64_t T, int64_t K, int group);
cudaError_t launch_decode_gemm(const DecodeArgs& a, int nsm, cudaStream_t st);

cudaError_t launch_relayout_shards(const void* src, void* dst, int64_t T, int64_t n_shard, int world,
                                   int64_t ldy, int elem_bytes, cudaStream_t st);

}  // namespace rrs

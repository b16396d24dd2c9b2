// C-ABI host layer of librrs (include/rrs.h): validation, workspace carving, launches, NCCL comm.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/rrs.h"
#include "kernels.h"

namespace {

thread_local std::string g_last_error;

rrs_status fail(rrs_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
rrs_status fail(rrs_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

rrs_status cuda_fail(cudaError_t e, const char* what) {
  return fail(RRS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

struct DevInfo {
  int major = 0, minor = 0, nsm = 0;
};

// per-device cached properties
DevInfo device_info(int& dev, cudaError_t& err) {
  static std::mutex mu;
  static DevInfo cache[64];
  static bool have[64] = {};
  err = cudaGetDevice(&dev);
  if (err != cudaSuccess || dev < 0 || dev >= 64) return DevInfo{};
  std::lock_guard<std::mutex> lk(mu);
  if (!have[dev]) {
    cudaDeviceProp p;
    err = cudaGetDeviceProperties(&p, dev);
    if (err != cudaSuccess) return DevInfo{};
    cache[dev].major = p.major;
    cache[dev].minor = p.minor;
    cache[dev].nsm = p.multiProcessorCount;
    have[dev] = true;
  }
  return cache[dev];
}

rrs_status check_arch(int& nsm) {
  int dev;
  cudaError_t e;
  DevInfo d = device_info(dev, e);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (d.major != 10 || d.minor != 0)
    return fail(RRS_ERR_ARCH, "device %d is sm_%d%d; librrs is built for sm_100a (B200) only", dev, d.major,
                d.minor);
  nsm = d.nsm;
  return RRS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Smoothing group: the paper's 128 = the GEMM K-block, and the Table-4 sizes; a power of
// two in [32, 1024] (a multiple of the 32-deep MMA K-step that divides or is divided by the 128-deep K-block)
// G = K / group is capped at kMaxGroups: the FP32 scale-accumulate sum_g fl(s_g rs) P_g has a worst-case
// normalised error of about (G + 2) 2^-24, which stays under the north_star's 1e-5 only for
// G <= 165; beyond that the parity bar could not be promised, so such calls are refused.
constexpr int64_t kMaxGroups = 160;

rrs_status check_group(int64_t K, int32_t group) {
  if (group < 32 || group > 1024 || (group & (group - 1)))
    return fail(RRS_ERR_INVALID_ARGUMENT, "group=%d: need a power of two in [32, 1024] (128 = P:189)", group);
  if (K <= 0 || K % group || K % 128)
    return fail(RRS_ERR_UNSUPPORTED_SHAPE, "K=%lld must be a positive multiple of group %d and of 128", (long long)K, group);
  if (K / group > kMaxGroups)
    return fail(RRS_ERR_UNSUPPORTED_SHAPE, "K/group = %lld groups > %lld: the 1e-5 FP32 bound needs G <= 160 (DESIGN.md §5)",
                (long long)(K / group), (long long)kMaxGroups);
  return RRS_OK;
}

rrs_status check_shape(int64_t T, int64_t K, int32_t group) {
  if (T < 0) return fail(RRS_ERR_INVALID_ARGUMENT, "T=%lld < 0", (long long)T);
  if (rrs_status s = check_group(K, group)) return s;
  if (!rrs::prologue_supports_k(K))
    return fail(RRS_ERR_UNSUPPORTED_SHAPE, "K=%lld: need 2^m in [128,16384] or 28*2^m in {7168,14336}", (long long)K);
  return RRS_OK;
}

struct Workspace {
  float* Xr;        // rotated activation X~ f32 [T][K] (written once by the FWHT pass, read by the quant pass)
  float* chan_max;
  float* s_group;
  float* x_scale;
  int8_t* Xq8;
  void* y_shard;
  void* y_gather;
  float* part;      // split-K partials f32 [kMaxSplits][T][N] (decode-sized T only)
};
constexpr int kMaxSplits = 8;
constexpr int64_t kSplitMaxT = 128;  // the single-CTA (M = 128) GEMM regime

// gather_world: ranks of the column-parallel communicator whose shard / gather buffers are carved (0 = none)
size_t carve(void* base, int64_t T, int64_t N, int64_t K, int32_t group, int32_t gather_world, Workspace* w) {
  const int32_t world = gather_world;
  size_t off = 0;
  auto take = [&](size_t bytes) -> void* {
    void* p = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(bytes);
    return p;
  };
  Workspace tmp;
  Workspace& ws = w ? *w : tmp;
  ws.Xr = static_cast<float*>(take(sizeof(float) * (size_t)T * K));
  ws.chan_max = static_cast<float*>(take(sizeof(float) * K));
  ws.s_group = static_cast<float*>(take(sizeof(float) * (K / group)));
  ws.x_scale = static_cast<float*>(take(sizeof(float) * (T > 0 ? T : 1)));
  ws.Xq8 = static_cast<int8_t*>(take((size_t)T * K));
  ws.y_shard = nullptr;
  ws.y_gather = nullptr;
  // split-K partials only where choose_splits can pick more than one split: decode-sized T, no communicator, N % 4 == 0
  // and few enough 240-column tiles that two splits of each fit on the GPU (<= 160 SMs on any sm_100 part); otherwise
  // (e.g. T = 128, N = 28672) the 8 T N floats would be dead scratch
  const bool split_ok = T > 0 && T <= kSplitMaxT && world == 0 && N % 4 == 0 && (N + 239) / 240 * 2 <= 160;
  ws.part = split_ok ? static_cast<float*>(take(sizeof(float) * kMaxSplits * (size_t)T * N)) : nullptr;
  if (world >= 1) {
    const int64_t ns = N / world;
    ws.y_shard = take((size_t)T * ns * 4);
    ws.y_gather = take((size_t)T * N * 4);
  }
  return off;
}

}  // namespace

struct rrs_comm_s {
  ncclComm_t nccl;
  int rank, world;
  cudaStream_t side = nullptr;  // all-gather + relayout of GEMM token slabs, overlapping the next slab's GEMM
  cudaEvent_t ev[9] = {};       // [0..7] slab GEMM done, [8] side stream done
};
constexpr int kMaxSlabs = 8;
constexpr int kNcclCtas = 16;  // SMs left to NCCL while a slab GEMM runs

static rrs_status gather_columns(const void* shard, int64_t T, int64_t N_total, int esz, void* Y, int64_t ldy,
                                 rrs_comm_t comm, void* gather_buf, cudaStream_t st) {
  const int world = comm->world;
  const int64_t n_local = N_total / world;
  if ((n_local * esz) % 16 || (ldy * esz) % 16)
    return fail(RRS_ERR_MISALIGNED, "shard width and ldy must be multiples of 16 bytes");
  ncclResult_t r = ncclAllGather(shard, gather_buf, (size_t)T * n_local * esz, ncclUint8, comm->nccl, st);
  if (r != ncclSuccess) return fail(RRS_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  cudaError_t e = rrs::launch_relayout_shards(gather_buf, Y, T, n_local, world, ldy, esz, st);
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "relayout kernel");
}


namespace rrs {
cudaError_t prepare_kernel_impl(const void* fn, int smem, int threads, int* blocks_per_sm) {
  static std::mutex mu;
  static KernelPrep cache[256];
  static int n = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < n; ++i) {
    if (cache[i].fn == fn && cache[i].dev == dev) {
      if (blocks_per_sm) *blocks_per_sm = cache[i].per_sm;
      return cudaSuccess;
    }
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  if (n < 256) cache[n++] = KernelPrep{fn, dev, per_sm};
  if (blocks_per_sm) *blocks_per_sm = per_sm;
  return cudaSuccess;
}
int max_active_clusters_impl(const void* fn, int cluster, int threads, int smem) {
  static std::mutex mu;
  struct Entry { const void* fn; int dev, n; };
  static Entry cache[128];
  static int n = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < n; ++i)
    if (cache[i].fn == fn && cache[i].dev == dev) return cache[i].n;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 1024);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  int c = 0;
  if (cudaOccupancyMaxActiveClusters(&c, fn, &cfg) != cudaSuccess || c < 1) {
    cudaGetLastError();
    c = 0;
  }
  if (n < 128) cache[n++] = Entry{fn, dev, c};
  return c;
}
}  // namespace rrs

extern "C" {

const char* rrs_status_str(int s) {
  switch (s) {
    case RRS_OK: return "RRS_OK";
    case RRS_ERR_INVALID_ARGUMENT: return "RRS_ERR_INVALID_ARGUMENT";
    case RRS_ERR_UNSUPPORTED_SHAPE: return "RRS_ERR_UNSUPPORTED_SHAPE";
    case RRS_ERR_MISALIGNED: return "RRS_ERR_MISALIGNED";
    case RRS_ERR_WORKSPACE_TOO_SMALL: return "RRS_ERR_WORKSPACE_TOO_SMALL";
    case RRS_ERR_ARCH: return "RRS_ERR_ARCH";
    case RRS_ERR_CUDA: return "RRS_ERR_CUDA";
    case RRS_ERR_NCCL: return "RRS_ERR_NCCL";
    default: return "RRS_ERR_UNKNOWN";
  }
}

const char* rrs_last_error(void) { return g_last_error.c_str(); }

int rrs_version(void) { return 102; }

size_t rrs_workspace_bytes(int64_t T, int64_t N, int64_t K, int32_t group, int32_t world) {
  if (T < 0 || K <= 0 || group <= 0 || K % group || world < 1 || (world > 1 && (N <= 0 || N % world))) return 0;
  return carve(nullptr, T, N, K, group, world > 1 ? world : 0, nullptr);
}

size_t rrs_workspace_bytes_comm(int64_t T, int64_t N, int64_t K, int32_t group, int32_t world) {
  if (T < 0 || K <= 0 || group <= 0 || K % group || world < 1 || N <= 0 || N % world) return 0;
  return carve(nullptr, T, N, K, group, world, nullptr);
}

rrs_status rrs_perm_from_channel_max(const float* chan_max, int64_t K, int32_t* perm, void* stream) {
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (!chan_max || !perm) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (K <= 0 || K > 16384) return fail(RRS_ERR_UNSUPPORTED_SHAPE, "K=%lld out of range", (long long)K);
  cudaError_t e = rrs::launch_perm_rank(chan_max, K, perm, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "perm_rank_kernel");
}

rrs_status rrs_prepare_weights(const void* W, int32_t w_dtype, int64_t N, int64_t K, int32_t group,
                               const int32_t* perm, uint8_t* Wq, uint8_t* Wop, float* w_scale, uint32_t flags,
                               void* stream) {
  int8_t* Wq8 = reinterpret_cast<int8_t*>(Wop);
  const bool e4m3 = (flags & RRS_OPERAND_I8) == 0;
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (w_dtype != RRS_BF16) return fail(RRS_ERR_INVALID_ARGUMENT, "W must be bf16 (R17)");
  if (N < 1) return fail(RRS_ERR_INVALID_ARGUMENT, "N=%lld < 1", (long long)N);
  if (rrs_status s = check_shape(N, K, group)) return s;
  if (!W || !perm || !w_scale || (!Wq && !Wq8)) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  const bool dec4 = (flags & RRS_W_PACKED4) != 0;  // Wop = decode4-packed [N][K/2] instead of bytes [N][K]
  if (!aligned16(W) || !aligned16(perm) || !aligned16(Wq) || !aligned16(Wq8))
    return fail(RRS_ERR_MISALIGNED, "pointers must be 16-byte aligned");
  // offline path: rotate a chunk of rows into a stream-ordered temporary, then quantise it per row
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(N, (int64_t(256) << 20) / (K * 4)));
  float* tmp = nullptr;
  cudaError_t e = cudaSuccess;
  if (dec4 && Wq8)  // the decode4 tiles cover ceil(N/256)*256 rows: the padding rows are zero codes
    e = cudaMemsetAsync(Wop, 0, (size_t)((N + 255) / 256) * 256 * (K / 2), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync (decode4 padding)");
  e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(float) * chunk * K, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (weight rotation scratch)");
  const uint16_t* Wb = static_cast<const uint16_t*>(W);
  for (int64_t n0 = 0; n0 < N && e == cudaSuccess; n0 += chunk) {
    const int64_t rows = std::min(chunk, N - n0);
    e = (flags & RRS_NO_ROTATION) ? rrs::launch_convert_colmax(Wb + n0 * K, rows, K, nullptr, tmp, nsm, st)
                                  : rrs::launch_fwht_colmax(Wb + n0 * K, rows, K, nullptr, tmp, nsm, st);
    if (e == cudaSuccess && (Wq || !dec4))
      e = rrs::launch_smooth_quant(tmp, rows, K, perm, nullptr, nullptr, Wq ? Wq + n0 * (K / 2) : nullptr,
                                   (Wq8 && !dec4) ? Wq8 + n0 * K : nullptr, w_scale + n0, e4m3, 128, nsm, st);
    if (e == cudaSuccess && Wq8 && dec4)  // the decode4 packing of the same codes (same kernel, other layout)
      e = rrs::launch_smooth_quant(tmp, rows, K, perm, nullptr, nullptr, Wop + n0 * (K / 2), nullptr, w_scale + n0,
                                   e4m3, 128, nsm, st, true);
  }
  cudaError_t e2 = cudaFreeAsync(tmp, st);
  if (e != cudaSuccess) return cuda_fail(e, "weight preparation kernels");
  return e2 == cudaSuccess ? RRS_OK : cuda_fail(e2, "cudaFreeAsync");
}

// rows a1-a6 (rotate = a1 on, smooth = a2-a5 on; the variants are rrs.h RRS_NO_ROTATION / RRS_PREROTATED and the
// RRS_NO_SMOOTH efficiency baselines)
static rrs_status prologue(const void* X, int64_t T, int64_t K, const int32_t* perm, uint8_t* Xq, int8_t* Xq8,
                           float* x_scale, float* s_group, float* chan_max, bool want_chan_max, float* Xr, bool e4m3,
                           int group, int nsm, cudaStream_t st, bool rotate = true, bool smooth = true) {
  if (!rotate || !smooth) {  // variant prologue: two kernels
    cudaError_t e = cudaSuccess;
    if (smooth) e = cudaMemsetAsync(chan_max, 0, sizeof(float) * K, st);
    unsigned* cm = smooth ? reinterpret_cast<unsigned*>(chan_max) : nullptr;
    const uint16_t* Xb = static_cast<const uint16_t*>(X);
    if (e == cudaSuccess)
      e = rotate ? rrs::launch_fwht_colmax(Xb, T, K, cm, Xr, nsm, st) : rrs::launch_convert_colmax(Xb, T, K, cm, Xr, nsm, st);
    if (e == cudaSuccess)
      e = rrs::launch_smooth_quant(Xr, T, K, perm, cm, s_group, Xq, Xq8, x_scale, e4m3, group, nsm, st);
    return e == cudaSuccess ? RRS_OK : cuda_fail(e, "variant prologue kernels");
  }
  if (T > 0 && rrs::prologue_decode_supports(T, K, group)) {  // decode-sized T: one launch, no memset
    // (without a chan_max output: the group-max variant, one grid barrier and no per-channel maxima)
    cudaError_t e = rrs::launch_prologue_decode(static_cast<const uint16_t*>(X), T, K, perm,
                                                want_chan_max ? reinterpret_cast<unsigned*>(chan_max) : nullptr, Xr,
                                                s_group, Xq, Xq8, x_scale, e4m3, group, st);
    return e == cudaSuccess ? RRS_OK : cuda_fail(e, "prologue_decode_kernel");
  }
  // prefill, K = 2^m: one cooperative launch that reduces group maxima only (s_g needs no per-channel c_j); a caller
  // that wants chan_max, or a grid that cannot be co-resident, takes the two-kernel prologue below
  cudaError_t e = cudaSuccess;
  // (only while X~ stays L2-resident: at 8192 x 8192 the fused kernel's second pass re-reads 268 MB from HBM and the
  // two-kernel path, which streams it once in a pass sized for that, is faster: 218 vs 258 us, profiles/time_prologue)
  if (T > 0 && !want_chan_max && rrs::prologue_fused_supports_k(K) && T * K * 4 <= (int64_t(80) << 20)) {
    e = rrs::launch_prologue_fused(static_cast<const uint16_t*>(X), T, K, Xr, perm, s_group, Xq, Xq8, x_scale, e4m3,
                                   group, st);
    if (e == cudaSuccess) return RRS_OK;
    if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported)
      return cuda_fail(e, "prologue_group_kernel");
    cudaGetLastError();
  }
  e = cudaMemsetAsync(chan_max, 0, sizeof(float) * K, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(chan_max)");
  e = rrs::launch_fwht_colmax(static_cast<const uint16_t*>(X), T, K, reinterpret_cast<unsigned*>(chan_max), Xr,
                              nsm, st);
  if (e != cudaSuccess) return cuda_fail(e, "fwht_colmax_kernel");
  e = rrs::launch_smooth_quant(Xr, T, K, perm, reinterpret_cast<const unsigned*>(chan_max), s_group, Xq, Xq8,
                               x_scale, e4m3, group, nsm, st);
  if (e != cudaSuccess) return cuda_fail(e, "smooth_quant_kernel");
  return RRS_OK;
}

rrs_status rrs_rotate_smooth_quant(const void* X, int32_t x_dtype, int64_t T, int64_t K, int32_t group,
                                   const int32_t* perm, uint8_t* Xq, uint8_t* Xop, float* x_scale, float* s_group,
                                   float* chan_max, void* ws, size_t ws_bytes, uint32_t flags, void* stream) {
  int8_t* Xq8 = reinterpret_cast<int8_t*>(Xop);
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (x_dtype != RRS_BF16) return fail(RRS_ERR_INVALID_ARGUMENT, "X must be bf16 (R17)");
  if (rrs_status s = check_shape(T, K, group)) return s;
  if ((T > 0 && !X) || !perm || !s_group || (T > 0 && !x_scale))
    return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!aligned16(X) || !aligned16(perm) || !aligned16(Xq) || !aligned16(Xq8))
    return fail(RRS_ERR_MISALIGNED, "pointers must be 16-byte aligned");
  Workspace w;
  const size_t need = carve(ws, T, 1, K, group, 0, &w);
  if (!ws || ws_bytes < need) return fail(RRS_ERR_WORKSPACE_TOO_SMALL, "need %zu workspace bytes", need);
  if (!aligned16(ws)) return fail(RRS_ERR_MISALIGNED, "workspace must be 16-byte aligned");
  const bool want_chan_max = chan_max != nullptr;
  if (!chan_max) chan_max = w.chan_max;
  return prologue(X, T, K, perm, Xq, Xq8, x_scale, s_group, chan_max, want_chan_max, w.Xr,
                  (flags & RRS_OPERAND_I8) == 0, group, nsm, static_cast<cudaStream_t>(stream),
                  (flags & (RRS_NO_ROTATION | RRS_PREROTATED)) == 0, (flags & RRS_NO_SMOOTH) == 0);
}

static rrs_status gemm_checks(const int8_t* Xq8, const float* x_scale, const int8_t* Wq8, const float* w_scale,
                              int64_t T, int64_t N, int64_t K, int32_t group, const void* Y, int64_t ldy,
                              bool swiglu = false) {
  if (swiglu && N % 2) return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_GEMM_SWIGLU needs an even N (gate/up pairs)");
  const int64_t n_out = swiglu ? N / 2 : N;
  if (T < 0 || N < 1) return fail(RRS_ERR_INVALID_ARGUMENT, "T=%lld N=%lld", (long long)T, (long long)N);
  if (rrs_status s = check_group(K, group)) return s;
  if (T > 0 && (!Xq8 || !x_scale || !Y)) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (!Wq8 || !w_scale) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (ldy < n_out) return fail(RRS_ERR_INVALID_ARGUMENT, "ldy=%lld < %lld output columns", (long long)ldy, (long long)n_out);
  if (!aligned16(Xq8) || !aligned16(Wq8) || !aligned16(Y) || ldy % 8)
    return fail(RRS_ERR_MISALIGNED, "pointers 16-byte aligned and ldy %% 8 == 0 required");
  return RRS_OK;
}

rrs_status rrs_gemm(const uint8_t* Xop, const float* x_scale, const float* s_group, const uint8_t* Wop,
                    const float* w_scale, int64_t T, int64_t N, int64_t K, int32_t group, float out_scale,
                    uint32_t flags, void* Y, int32_t y_dtype, int64_t ldy, void* stream) {
  const int8_t* Xq8 = reinterpret_cast<const int8_t*>(Xop);
  const int8_t* Wq8 = reinterpret_cast<const int8_t*>(Wop);
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  const bool swiglu = (flags & RRS_GEMM_SWIGLU) != 0;
  if (rrs_status s = gemm_checks(Xq8, x_scale, Wq8, w_scale, T, N, K, group, Y, ldy, swiglu)) return s;
  if (flags & RRS_W_PACKED4) {
    if (flags & (RRS_GEMM_PLAIN | RRS_GEMM_SWIGLU | RRS_GEMM_SUBCHANNEL))
      return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_W_PACKED4: no PLAIN / SWIGLU / SUBCHANNEL");
    if (!s_group) return fail(RRS_ERR_INVALID_ARGUMENT, "s_group is NULL");
    if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
    if (T == 0) return RRS_OK;
    if (!rrs::decode_gemm_supports(T, K, group))
      return fail(RRS_ERR_UNSUPPORTED_SHAPE, "RRS_W_PACKED4: 1 <= T <= 64 and group %% 128 == 0 (T=%lld, group=%d)",
                  (long long)T, group);
    rrs::DecodeArgs d{Xq8, x_scale, s_group, Wop, w_scale, T, N, K, group, out_scale, Y, y_dtype, ldy};
    cudaError_t e = rrs::launch_decode_gemm(d, nsm, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_decode_gemm kernel");
  }
  const bool plain = (flags & RRS_GEMM_PLAIN) != 0;
  const bool sub = (flags & RRS_GEMM_SUBCHANNEL) != 0;
  if (sub && (plain || swiglu || (flags & RRS_OPERAND_I8) || N % 8 || !aligned16(w_scale)))
    return fail(RRS_ERR_INVALID_ARGUMENT,
                "RRS_GEMM_SUBCHANNEL: E4M3 operands, N %% 8 == 0, 16-byte aligned scales, no PLAIN / SWIGLU");
  if (swiglu && (plain || y_dtype != RRS_BF16))
    return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_GEMM_SWIGLU: bf16 output of the RRS (not plain) GEMM only");
  if (!plain && !sub && !s_group) return fail(RRS_ERR_INVALID_ARGUMENT, "s_group is NULL");
  if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
  if (T == 0) return RRS_OK;
  rrs::GemmArgs a{Xq8, x_scale, s_group, Wq8, w_scale, T, N, K, group, out_scale, plain,
                  (flags & RRS_OPERAND_I8) == 0, Y, y_dtype, ldy, nullptr, swiglu};
  a.subchannel = sub;
  cudaError_t e = rrs::launch_gemm(a, nsm, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_gemm kernel");
}

// Decode-sized T (one M = 128 row block): the (T, N) tile grid covers only N/240 SMs, so the K range is split
// over up to kMaxSplits CTAs per tile (whole groups each) and a fixed-order reduction sums the f32 partials.
static int choose_splits(int64_t T, int64_t N, int64_t K, int32_t group, int nsm, const float* part) {
  if (!part || T > kSplitMaxT || N % 4) return 1;
  const int64_t tiles = (N + 239) / 240, KB = K / 128, G = K / group;
  int best = 1;
  for (int s = 2; s <= kMaxSplits; ++s)
    if (KB % s == 0 && G % s == 0 && tiles * s <= nsm) best = s;
  return best;
}

// The layer's GEMM, split-K when it pays (then Y is written by the reduction kernel).
static cudaError_t layer_gemm(rrs::GemmArgs a, const Workspace& w, int nsm, cudaStream_t st) {
  const int splits = a.swiglu ? 1 : choose_splits(a.T, a.N, a.K, a.group, nsm, w.part);
  if (splits == 1) return rrs::launch_gemm(a, nsm, st);
  void* Y = a.Y;
  const int y_dtype = a.y_dtype;
  const int64_t ldy = a.ldy;
  a.splits = splits;
  a.Y = w.part;
  a.y_dtype = 1;
  a.ldy = a.N;
  cudaError_t e = rrs::launch_gemm(a, nsm, st);
  if (e != cudaSuccess) return e;
  return rrs::launch_reduce_splits(w.part, splits, a.T, a.N, Y, y_dtype, ldy, st);
}

// token-sharded data parallel.  The prologue runs as its two passes (the fused single-kernel
// prologue has a grid barrier where the cross-rank reduction must go): rotate + local channel max, one
// ncclAllReduce(MAX) of chan_max[K] (non-negative floats: max is exact and order-free), smooth + quantise.
static rrs_status linear_token_sharded(const void* X, int64_t T, int64_t K, int32_t group, const int32_t* perm,
                                       const int8_t* Wq8, const float* w_scale, int64_t N, void* Y, int32_t y_dtype,
                                       int64_t ldy, rrs_comm_t comm, void* ws, size_t ws_bytes, bool e4m3,
                                       bool swiglu, int nsm, cudaStream_t st) {
  if (N < 1) return fail(RRS_ERR_INVALID_ARGUMENT, "N_total=%lld < 1", (long long)N);
  if ((T > 0 && !X) || !perm) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
  Workspace w;
  const size_t need = carve(ws, T, N, K, group, 0, &w);
  if (!ws || ws_bytes < need) return fail(RRS_ERR_WORKSPACE_TOO_SMALL, "need %zu workspace bytes", need);
  if (!aligned16(X) || !aligned16(perm) || !aligned16(ws)) return fail(RRS_ERR_MISALIGNED, "16-byte alignment");
  if (T > 0)
    if (rrs_status s = gemm_checks(w.Xq8, w.x_scale, Wq8, w_scale, T, N, K, group, Y, ldy, swiglu)) return s;
  cudaError_t e = cudaMemsetAsync(w.chan_max, 0, sizeof(float) * K, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(chan_max)");
  e = rrs::launch_fwht_colmax(static_cast<const uint16_t*>(X), T, K, reinterpret_cast<unsigned*>(w.chan_max), w.Xr,
                              nsm, st);
  if (e != cudaSuccess) return cuda_fail(e, "fwht_colmax_kernel");
  ncclResult_t r = ncclAllReduce(w.chan_max, w.chan_max, (size_t)K, ncclFloat, ncclMax, comm->nccl, st);
  if (r != ncclSuccess) return fail(RRS_ERR_NCCL, "ncclAllReduce(chan_max, MAX): %s", ncclGetErrorString(r));
  if (T == 0) return RRS_OK;
  e = rrs::launch_smooth_quant(w.Xr, T, K, perm, reinterpret_cast<const unsigned*>(w.chan_max), w.s_group, nullptr,
                               w.Xq8, w.x_scale, e4m3, group, nsm, st);
  if (e != cudaSuccess) return cuda_fail(e, "smooth_quant_kernel");
  rrs::GemmArgs a{w.Xq8, w.x_scale, w.s_group, Wq8, w_scale, T, N, K, group, 1.0f / (float)K, false, e4m3, Y,
                  y_dtype, ldy, nullptr, swiglu};
  e = layer_gemm(a, w, nsm, st);
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_gemm kernel");
}

rrs_status rrs_linear(const void* X, int32_t x_dtype, int64_t T, int64_t K, int32_t group, const int32_t* perm,
                      const uint8_t* Wop, const float* w_scale, int64_t N_total, void* Y, int32_t y_dtype,
                      int64_t ldy, rrs_comm_t comm, void* ws, size_t ws_bytes, uint32_t flags, void* stream) {
  const int8_t* Wq8 = reinterpret_cast<const int8_t*>(Wop);
  const bool e4m3 = (flags & RRS_OPERAND_I8) == 0;
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (x_dtype != RRS_BF16) return fail(RRS_ERR_INVALID_ARGUMENT, "X must be bf16 (R17)");
  if (rrs_status s = check_shape(T, K, group)) return s;
  const bool swiglu = (flags & RRS_GEMM_SWIGLU) != 0;
  if (swiglu && y_dtype != RRS_BF16) return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_GEMM_SWIGLU: bf16 output only");
  const bool rotate = (flags & (RRS_NO_ROTATION | RRS_PREROTATED)) == 0, smooth = (flags & RRS_NO_SMOOTH) == 0;
  if ((flags & RRS_NO_ROTATION) && (flags & RRS_PREROTATED))
    return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_NO_ROTATION and RRS_PREROTATED are exclusive");
  if ((!rotate || !smooth) && comm && (flags & RRS_TOKEN_SHARDED))
    return fail(RRS_ERR_INVALID_ARGUMENT, "prologue variants are not supported with RRS_TOKEN_SHARDED");
  // R1: (1/sqrt K)^2 when the Hadamard rotation is in the layer (online or pre-applied), exact for K = 2^m
  const float out_scale = (flags & RRS_NO_ROTATION) ? 1.0f : 1.0f / (float)K;
  if (flags & RRS_W_PACKED4) {  // decode regime: int8 activation codes + the packed-W stream (decode.cu)
    if (comm || swiglu) return fail(RRS_ERR_INVALID_ARGUMENT, "RRS_W_PACKED4: single GPU, no SWIGLU");
    if (T > 0 && !rrs::decode_gemm_supports(T, K, group))
      return fail(RRS_ERR_UNSUPPORTED_SHAPE, "RRS_W_PACKED4: 1 <= T <= 64 and group %% 128 == 0 (T=%lld, group=%d)",
                  (long long)T, group);
    if (N_total < 1) return fail(RRS_ERR_INVALID_ARGUMENT, "N_total=%lld < 1", (long long)N_total);
    if ((T > 0 && !X) || !perm) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
    if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
    Workspace w;
    const size_t need = carve(ws, T, N_total, K, group, 0, &w);
    if (!ws || ws_bytes < need) return fail(RRS_ERR_WORKSPACE_TOO_SMALL, "need %zu workspace bytes", need);
    if (!aligned16(X) || !aligned16(perm) || !aligned16(ws)) return fail(RRS_ERR_MISALIGNED, "16-byte alignment");
    if (T > 0)
      if (rrs_status s = gemm_checks(w.Xq8, w.x_scale, Wq8, w_scale, T, N_total, K, group, Y, ldy)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (rrs_status s = prologue(X, T, K, perm, nullptr, w.Xq8, w.x_scale, w.s_group, w.chan_max, false, w.Xr,
                                /*e4m3=*/false, group, nsm, st, rotate, smooth))
      return s;
    if (T == 0) return RRS_OK;
    rrs::DecodeArgs d{w.Xq8, w.x_scale, w.s_group, Wop, w_scale, T, N_total, K, group, out_scale, Y, y_dtype, ldy};
    cudaError_t e = rrs::launch_decode_gemm(d, nsm, st);
    return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_decode_gemm kernel");
  }
  if (comm && (flags & RRS_TOKEN_SHARDED))
    return linear_token_sharded(X, T, K, group, perm, Wq8, w_scale, N_total, Y, y_dtype, ldy, comm, ws, ws_bytes, e4m3,
                                swiglu, nsm, static_cast<cudaStream_t>(stream));
  const int world = comm ? comm->world : 1;
  if (N_total < 1 || N_total % world)
    return fail(RRS_ERR_INVALID_ARGUMENT, "N_total=%lld must be a positive multiple of world=%d", (long long)N_total, world);
  const int64_t n_local = N_total / world;
  if ((T > 0 && !X) || !perm) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
  Workspace w;
  const size_t need = carve(ws, T, N_total, K, group, comm ? world : 0, &w);
  if (!ws || ws_bytes < need) return fail(RRS_ERR_WORKSPACE_TOO_SMALL, "need %zu workspace bytes", need);
  if (!aligned16(X) || !aligned16(perm) || !aligned16(ws)) return fail(RRS_ERR_MISALIGNED, "16-byte alignment");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int esz = y_dtype == RRS_F32 ? 4 : 2;
  // with the fused SwiGLU each rank's shard holds whole (gate, up) pairs and yields n_local / 2 outputs
  const int64_t n_out_local = swiglu ? n_local / 2 : n_local, n_out = swiglu ? N_total / 2 : N_total;
  // every argument is validated before anything is enqueued (rrs.h conventions)
  if (T > 0) {
    if (!comm) {
      if (rrs_status s = gemm_checks(w.Xq8, w.x_scale, Wq8, w_scale, T, N_total, K, group, Y, ldy, swiglu)) return s;
    } else {
      if (rrs_status s = gemm_checks(w.Xq8, w.x_scale, Wq8, w_scale, T, n_local, K, group, w.y_shard, n_out_local, swiglu))
        return s;
      if (ldy < n_out || !Y || !aligned16(Y)) return fail(RRS_ERR_INVALID_ARGUMENT, "Y / ldy");
      if ((n_out_local * esz) % 16 || (ldy * esz) % 16)
        return fail(RRS_ERR_MISALIGNED, "shard width and ldy must be multiples of 16 bytes");
    }
  }
  if (rrs_status s = prologue(X, T, K, perm, nullptr, w.Xq8, w.x_scale, w.s_group, w.chan_max, false, w.Xr, e4m3,
                              group, nsm, st, rotate, smooth))
    return s;
  if (T == 0) return RRS_OK;
  if (!comm) {
    rrs::GemmArgs a{w.Xq8, w.x_scale, w.s_group, Wq8, w_scale, T, N_total, K, group, out_scale, false, e4m3, Y,
                    y_dtype, ldy, nullptr, swiglu};
    cudaError_t e = layer_gemm(a, w, nsm, st);
    return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_gemm kernel");
  }
  // column-parallel: local shard [T][n_local] -> all-gather [world][T][n_local] -> Y[T][ldy]
  // Token slabs (SURVEY §8(e) "overlap by token slabs"): the GEMM of slab s runs on `st` while the all-gather
  // and relayout of slab s-1 run on the communicator's side stream, so the NVLink transfer overlaps compute.
  // Slabs are whole 256-row M-blocks of the pair GEMM; the shard / gather buffers are laid out slab-major.
  // Slabs only while each slab's GEMM still fills the SMs it may use (pair tiles of 256 x 240 >= the pairs left
  // after kNcclCtas): at P = 8 on the C3 up shard (1792 columns) a quarter slab would fill only a third of them.
  const int64_t n_tiles = (n_local + 239) / 240, m_tiles = (T + 255) / 256;
  const int64_t pairs = (nsm - kNcclCtas) / 2;
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(4, (m_tiles * n_tiles) / std::max<int64_t>(1, pairs)));
  const int64_t rows = want > 1 ? ((m_tiles + want - 1) / want) * 256 : T;
  const int nslab = (int)((T + rows - 1) / rows);
  if (nslab > kMaxSlabs) return fail(RRS_ERR_INVALID_ARGUMENT, "too many slabs");
  cudaError_t e = cudaEventRecord(comm->ev[8], st);  // the side stream starts after the prologue (and whatever
  if (e == cudaSuccess) e = cudaStreamWaitEvent(comm->side, comm->ev[8], 0);  // came before it on st)
  if (e != cudaSuccess) return cuda_fail(e, "slab pipeline ordering");
  rrs_status status = RRS_OK;
  for (int sl = 0; sl < nslab && status == RRS_OK; ++sl) {
    const int64_t t0 = sl * rows, ts = std::min(rows, T - t0);
    char* shard = static_cast<char*>(w.y_shard) + t0 * n_out_local * esz;
    rrs::GemmArgs a{w.Xq8 + t0 * K, w.x_scale + t0, w.s_group, Wq8, w_scale, ts, n_local, K, group, out_scale, false,
                    e4m3, shard, y_dtype, n_out_local, nullptr, swiglu};
    e = rrs::launch_gemm(a, nslab > 1 ? nsm - kNcclCtas : nsm, st);  // leave SMs to the overlapping all-gather
    if (e != cudaSuccess) { status = cuda_fail(e, "rrs_gemm kernel"); break; }
    e = cudaEventRecord(comm->ev[sl], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(comm->side, comm->ev[sl], 0);
    if (e != cudaSuccess) { status = cuda_fail(e, "slab event"); break; }
    status = gather_columns(shard, ts, n_out, esz, static_cast<char*>(Y) + t0 * ldy * esz, ldy, comm,
                            static_cast<char*>(w.y_gather) + t0 * n_out * esz, comm->side);
  }
  // join the side stream on every path (also after an error: a capture must not end with it forked)
  e = cudaEventRecord(comm->ev[8], comm->side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, comm->ev[8], 0);  // Y complete in stream order on st
  if (status != RRS_OK) return status;
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "slab pipeline join");
}

rrs_status rrs_allgather_columns(const void* Y_shard, int64_t T, int64_t N_total, int32_t y_dtype, void* Y,
                                 int64_t ldy, rrs_comm_t comm, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (!comm) return fail(RRS_ERR_INVALID_ARGUMENT, "comm is NULL");
  if (y_dtype != RRS_BF16 && y_dtype != RRS_F32) return fail(RRS_ERR_INVALID_ARGUMENT, "y_dtype");
  if (T < 0 || N_total < 1 || N_total % comm->world || ldy < N_total)
    return fail(RRS_ERR_INVALID_ARGUMENT, "shape");
  if (T == 0) return RRS_OK;
  if (!Y_shard || !Y || !aligned16(Y_shard) || !aligned16(Y) || !aligned16(ws))
    return fail(RRS_ERR_MISALIGNED, "pointers");
  Workspace w;
  // any K with a valid carve works: the gather buffer only depends on T and N
  const size_t need = carve(ws, T, N_total, 128, 128, comm->world, &w);
  if (!ws || ws_bytes < need) return fail(RRS_ERR_WORKSPACE_TOO_SMALL, "need %zu workspace bytes", need);
  return gather_columns(Y_shard, T, N_total, y_dtype == RRS_F32 ? 4 : 2, Y, ldy, comm, w.y_gather,
                        static_cast<cudaStream_t>(stream));
}

rrs_status rrs_comm_unique_id(uint8_t id[128]) {
  g_last_error.clear();
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(RRS_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(id, &u, 128);
  return RRS_OK;
}

rrs_status rrs_comm_init(rrs_comm_t* comm, int32_t rank, int32_t world, const uint8_t id[128]) {
  g_last_error.clear();
  if (!comm || !id || world < 1 || rank < 0 || rank >= world) return fail(RRS_ERR_INVALID_ARGUMENT, "comm args");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  auto* c = new rrs_comm_s{};
  // NCCL kernels use at most kNcclCtas SMs; the slab GEMMs that overlap them leave that many SMs free (below), so
  // the all-gather of slab s really runs concurrently with the GEMM of slab s+1
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.maxCTAs = kNcclCtas;
  cfg.minCTAs = 1;
  ncclResult_t r = ncclCommInitRankConfig(&c->nccl, world, u, rank, &cfg);
  if (r != ncclSuccess) {
    delete c;
    return fail(RRS_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  c->rank = rank;
  c->world = world;
  cudaError_t e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  for (int i = 0; i < 9 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return cuda_fail(e, "side stream / events for the slab pipeline");
  }
  *comm = c;
  return RRS_OK;
}

rrs_status rrs_comm_destroy(rrs_comm_t comm) {
  g_last_error.clear();
  if (!comm) return RRS_OK;
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  for (int i = 0; i < 9; ++i)
    if (comm->ev[i]) cudaEventDestroy(comm->ev[i]);
  if (comm->side) cudaStreamDestroy(comm->side);
  delete comm;
  return r == ncclSuccess ? RRS_OK : fail(RRS_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
}

int32_t rrs_comm_world(rrs_comm_t comm) { return comm ? comm->world : 1; }
int32_t rrs_comm_rank(rrs_comm_t comm) { return comm ? comm->rank : 0; }

rrs_status rrs_debug_rotate(const void* X, int64_t T, int64_t K, float* Xr, float* chan_max, void* stream) {
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (rrs_status s = check_shape(T, K, 128)) return s;
  if (!chan_max || (T > 0 && (!X || !Xr))) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(chan_max, 0, sizeof(float) * K, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  e = rrs::launch_fwht_colmax(static_cast<const uint16_t*>(X), T, K, reinterpret_cast<unsigned*>(chan_max), Xr, nsm, st);
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "fwht_colmax_kernel");
}

rrs_status rrs_debug_relayout(const void* gathered, int64_t T, int64_t n_shard, int32_t world, int32_t y_dtype,
                              void* Y, int64_t ldy, void* stream) {
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (T < 0 || n_shard < 1 || world < 1 || ldy < n_shard * world || (y_dtype != RRS_BF16 && y_dtype != RRS_F32))
    return fail(RRS_ERR_INVALID_ARGUMENT, "shape");
  if (T == 0) return RRS_OK;
  const int esz = y_dtype == RRS_F32 ? 4 : 2;
  if (!gathered || !Y || !aligned16(gathered) || !aligned16(Y) || (n_shard * esz) % 16 || (ldy * esz) % 16)
    return fail(RRS_ERR_MISALIGNED, "16-byte aligned buffers, shard width and ldy required");
  cudaError_t e = rrs::launch_relayout_shards(gathered, Y, T, n_shard, world, ldy, esz, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "relayout_kernel");
}

rrs_status rrs_debug_group_partials(const uint8_t* Xop, const uint8_t* Wop, int64_t T, int64_t N, int64_t K,
                                    int32_t group, int32_t* P, uint32_t flags, void* stream) {
  const int8_t* Xq8 = reinterpret_cast<const int8_t*>(Xop);
  const int8_t* Wq8 = reinterpret_cast<const int8_t*>(Wop);
  g_last_error.clear();
  int nsm;
  if (rrs_status s = check_arch(nsm)) return s;
  if (!P) return fail(RRS_ERR_INVALID_ARGUMENT, "null pointer");
  // the GEMM needs valid scale pointers; partials do not depend on them: use a scratch Y in P's tail? No:
  // the debug launch passes P and a null Y; the kernel skips the Y store when Y == nullptr.
  if (T < 0 || N < 1) return fail(RRS_ERR_INVALID_ARGUMENT, "shape");
  if (rrs_status s = check_group(K, group)) return s;
  if (!aligned16(Xq8) || !aligned16(Wq8)) return fail(RRS_ERR_MISALIGNED, "alignment");
  if (T == 0) return RRS_OK;
  rrs::GemmArgs a{Xq8, nullptr, nullptr, Wq8, nullptr, T, N, K, group, 1.0f, false, (flags & RRS_OPERAND_I8) == 0,
                  nullptr, RRS_F32, N, P};
  cudaError_t e = rrs::launch_gemm(a, nsm, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RRS_OK : cuda_fail(e, "rrs_gemm kernel (debug partials)");
}

}  // extern "C"

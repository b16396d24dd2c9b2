// TMA ingress microbenchmark (decides the GEMM tiling): bytes/clk/SM that TMA can deliver
// into shared memory for 2-D boxes of [rows x 128 B] (SWIZZLE_128B), L2-resident source, in 3 modes:
//   0 unicast, every CTA reads its own slice;  1 unicast, all CTAs read the same slice at the same time;
//   2 multicast: clusters of C CTAs, each CTA loads 1/C of every box and multicasts it to the whole cluster.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2409_20361_b200/csrc/ptx.cuh"

using namespace rrs::ptx;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

constexpr int STAGES = 4;
constexpr int BOX_ROWS = 256;                 // 32 KiB per box
constexpr int BOX_BYTES = BOX_ROWS * 128;

__device__ __forceinline__ void tma_mc(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1),
      "r"(smem_u32(bar)), "h"(mask) : "memory");
}

template <int C>
__global__ void tma_kernel(const __grid_constant__ CUtensorMap tm, int mode, int iters, int slice_boxes,
                           unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + STAGES * BOX_BYTES);
  uint64_t* empty = full + STAGES;
  uint32_t rank = 0;
  if (C > 1) rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (C > 1) cluster_sync();
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int cid = mode == 1 ? 0 : (C > 1 ? blockIdx.x / C : blockIdx.x);
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) {
        mbar_wait(&full[s], ((i / STAGES) - 1) & 1);          // our copy of the box has landed
        for (uint32_t r = 0; r < (uint32_t)C; ++r) {           // tell every CTA of the cluster: slot free here
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(r));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
        mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);         // every CTA has freed slot s
      }
      mbar_arrive_expect_tx(&full[s], BOX_BYTES);
      const int row0 = (cid * slice_boxes + (i % slice_boxes)) * BOX_ROWS;
      if (C == 1) {
        tma_load_2d(buf + s * BOX_BYTES, &tm, &full[s], 0, row0, kEvictNormal);
      } else {
        constexpr int part = BOX_ROWS / C;
        // each CTA fetches rows [rank*part, (rank+1)*part) of the box and multicasts them to all C CTAs
        // (the per-load box is part rows: the tensor map is encoded with box height = part)
        tma_mc(buf + s * BOX_BYTES + rank * part * 128, &tm, &full[s], 0, row0 + rank * part, (uint16_t)((1u << C) - 1));
      }
    }
    for (int i = iters; i < iters + STAGES; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], ((i / STAGES) - 1) & 1);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (C > 1) cluster_sync();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int C>
static int run(const char* name, int mode, uint8_t* data, int64_t rows, int nsm, unsigned long long* dcyc, int clk_khz) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, (cuuint32_t)(BOX_ROWS / C)};
  cuuint32_t es[2] = {1, 1};
  if (enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, data, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int smem = STAGES * BOX_BYTES + 2048;
  auto k = tma_kernel<C>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 2000, slice_boxes = 8;  // 8 boxes x 32 KiB = 256 KiB per slice; 148 slices = 37 MiB (L2)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm / C * C);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) CK(cudaLaunchKernelEx(&cfg, k, tm, mode, iters, slice_boxes, dcyc));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, k, tm, mode, iters, slice_boxes, dcyc));
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  const int g = nsm / C * C;
  CK(cudaMemcpy(h, dcyc, sizeof(unsigned long long) * g, cudaMemcpyDeviceToHost));
  double mx = 0;
  for (int i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes_per_cta = (double)iters * BOX_BYTES;
  printf("%-34s C=%d  %7.1f B/clk/SM delivered  (%.2f TB/s into smem, %.2f TB/s from L2)\n", name, C,
         bytes_per_cta / mx, bytes_per_cta * g / (ms * 1e-3) / 1e12, bytes_per_cta * g / C / (ms * 1e-3) / 1e12);
  return 0;
}

int main() {
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int64_t rows = (int64_t)nsm * 8 * BOX_ROWS;
  uint8_t* data;
  CK(cudaMalloc(&data, rows * 128));
  CK(cudaMemset(data, 1, rows * 128));
  unsigned long long* dcyc;
  CK(cudaMalloc(&dcyc, 1024 * 8));
  run<1>("unicast, distinct slices", 0, data, rows, nsm, dcyc, clk);
  run<1>("unicast, same slice for all", 1, data, rows, nsm, dcyc, clk);
  run<2>("multicast cluster, distinct", 0, data, rows, nsm, dcyc, clk);
  run<4>("multicast cluster, distinct", 0, data, rows, nsm, dcyc, clk);
  run<8>("multicast cluster, distinct", 0, data, rows, nsm, dcyc, clk);
  return 0;
}

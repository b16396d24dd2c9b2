// Shared device macro for the RRS sm_100a kernels (product path; never includes oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define RRS_DEVICE __device__ __forceinline__

// Shared device helpers for the RRS sm_100a kernels (product path; never includes oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define RRS_DEVICE __device__ __forceinline__

namespace rrs {

// bf16 bits -> double, exactly, with integer ops only (no F2F): sign | (exp8 + 896) << 20 | mant7 << 13.
// bf16 subnormals take the (rare) conversion path; Inf/NaN are unsupported inputs (DESIGN.md §3 R17).
RRS_DEVICE double bf16_bits_to_double(uint32_t b) {
  uint32_t mag = b & 0x7FFFu;
  uint32_t hi;
  if (mag >= 0x80u) {
    hi = ((b & 0x8000u) << 16) | ((mag << 13) + (896u << 20));
  } else if (mag == 0u) {
    hi = (b & 0x8000u) << 16;
  } else {
    return (double)__uint_as_float(b << 16);
  }
  return __hiloint2double((int)hi, 0);
}

// Branch-free variant for the hot loop: exact for normal numbers and zeros; sets `sub` when b is a
// bf16 subnormal (the caller then redoes the conversion with bf16_bits_to_double).
RRS_DEVICE double bf16_bits_to_double_fast(uint32_t b, bool& sub) {
  const uint32_t mag = b & 0x7FFFu;
  const uint32_t hi = ((b & 0x8000u) << 16) | (mag ? (mag << 13) + (896u << 20) : 0u);
  sub |= (mag - 1u) < 0x7Fu;
  return __hiloint2double((int)hi, 0);
}

RRS_DEVICE uint32_t float_as_ordered(float f) { return __float_as_uint(f); }  // valid for f >= +0

RRS_DEVICE int lane_id() { return threadIdx.x & 31; }

}  // namespace rrs

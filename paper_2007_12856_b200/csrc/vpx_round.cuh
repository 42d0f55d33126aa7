// Round-to-nearest TF32 for values stored into frames that feed tensor-core
// MMAs.  The tensor core truncates fp32 operands to TF32 (biased toward zero,
// so errors add up layer after layer); storing values already rounded to the
// nearest TF32 makes the MMA exact on them and the rounding unbiased.
#pragma once
#include <cstdint>

#include "conv_simt.h"

namespace vpx {
__device__ __forceinline__ float tf32_rn(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
__device__ __forceinline__ float rnd(const Frame& f, float v) { return f.rnd ? tf32_rn(v) : v; }
__device__ __forceinline__ float4 rnd4(const Frame& f, float4 v) {
  if (!f.rnd) return v;
  return make_float4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
}
}  // namespace vpx

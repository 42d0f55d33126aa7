// Round-to-nearest TF32 for values stored into frames that feed tensor-core
// MMAs.  The tensor core truncates fp32 operands to TF32 (biased toward zero,
// so errors add up layer after layer); storing values already rounded to the
// nearest TF32 makes the MMA exact on them and the rounding unbiased.
#pragma once
#include <cstdint>

#include "conv_simt.h"

namespace vpx {
// Same result as cvt.rna.tf32.f32 (nearest, ties away from zero) for every
// non-NaN input, including the carry into the exponent and overflow to inf,
// in two integer instructions instead of cvt's finite-check sequence.
__device__ __forceinline__ float tf32_rn(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ float rnd(const Frame& f, float v) { return f.rnd ? tf32_rn(v) : v; }
__device__ __forceinline__ float4 rnd4(const Frame& f, float4 v) {
  if (!f.rnd) return v;
  return make_float4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
}
}  // namespace vpx

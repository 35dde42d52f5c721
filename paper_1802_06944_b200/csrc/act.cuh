// Fused activation of the forward epilogues (kernel.py activation set; softmax runs as a
// separate row kernel). ACT is a template parameter so each epilogue stays branch-free.
#pragma once

#include "../../include/deepthin_b200.h"

namespace dt {

template <int ACT>
__device__ __forceinline__ float act_apply(float z, float arg) {
  if constexpr (ACT == DT_ACT_RELU) return z > 0.f ? z : 0.f;
  if constexpr (ACT == DT_ACT_SIGMOID) return 1.f / (1.f + expf(-z));
  if constexpr (ACT == DT_ACT_TANH) return tanhf(z);
  if constexpr (ACT == DT_ACT_CLIPPED_RELU) return fminf(fmaxf(z, 0.f), arg);
  return z;
}

// Tensor-core-path epilogues: MUFU ex2 + rcp (__expf / __fdividef, absolute error ~1e-7 on
// the bounded outputs) instead of the accurate expf / tanhf / IEEE division sequences.
template <int ACT>
__device__ __forceinline__ float act_fast(float z, float arg) {
  if constexpr (ACT == DT_ACT_SIGMOID) return __fdividef(1.f, 1.f + __expf(-z));
  if constexpr (ACT == DT_ACT_TANH) return 1.f - __fdividef(2.f, 1.f + __expf(2.f * z));
  return act_apply<ACT>(z, arg);
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// bf16 outputs of the tensor-core path: one MUFU op per element for sigmoid / tanh
// (tanh.approx, relative error 2^-11: <= 2.5e-4 absolute on a sigmoid, below the bf16 output's
// own rounding of up to 2^-9 relative); fp32 outputs: act_fast (ex2 + rcp, ~1e-7).
template <int YDT, int ACT>
__device__ __forceinline__ float act_out_bf16(float z, float arg) {
  if constexpr (YDT == DT_BF16 && ACT == DT_ACT_SIGMOID) return fmaf(0.5f, tanh_approx(0.5f * z), 0.5f);
  if constexpr (YDT == DT_BF16 && ACT == DT_ACT_TANH) return tanh_approx(z);
  return act_fast<ACT>(z, arg);
}

}  // namespace dt

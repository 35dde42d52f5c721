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

}  // namespace dt

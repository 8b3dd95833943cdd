// elem.cuh — per-element building blocks shared by the sm_100a kernels: the NaN-propagating max and
// the penalty formula in exactly specified binary32 arithmetic.
#pragma once
#include "common.cuh"

namespace smp {

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Penalised logit, every op correctly rounded binary32 with no FMA
// contraction (R1, R3): OPENAI_CTRL  y = x; if r != 1: y = y > 0 ? y/r : y*r;
// if cnt > 0: y -= freq*cnt; y -= pres.   LINEAR  y = ((x - freq*cnt) - pres*[cnt>0]) - rep.
__device__ __forceinline__ float apply_penalty(float x, uint32_t meta, const sampling_params& p, int mode) {
  const int cnt = (int)(meta >> 1);
  float y = x;
  if (mode == SAMPLER_PEN_OPENAI_CTRL) {
    const float r = p.repetition_penalty;
    if (r != 1.0f) y = (y > 0.0f) ? __fdiv_rn(y, r) : __fmul_rn(y, r);
    if (cnt > 0) {
      y = __fsub_rn(y, __fmul_rn(p.frequency_penalty, (float)cnt));
      y = __fsub_rn(y, p.presence_penalty);
    }
  } else {
    y = __fsub_rn(y, __fmul_rn(p.frequency_penalty, (float)cnt));
    y = __fsub_rn(y, cnt > 0 ? p.presence_penalty : 0.0f);
    y = __fsub_rn(y, p.repetition_penalty);
  }
  return y;
}

}  // namespace smp

// elem.cuh — per-element building blocks shared by the sm_100a kernels: 16-byte vector decode
// (bf16 / fp32), the penalty formula in exactly specified binary32 arithmetic, and the
// thread-private online softmax accumulator.
#pragma once
#include "common.cuh"

namespace smp {

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <typename T>
struct VecT;
template <>
struct VecT<__nv_bfloat16> {
  static constexpr int N = 8;
  // 8 logits from 16 bytes; vmax = NaN-propagating max (NaN / +inf detection for free)
  static __device__ __forceinline__ void load(const uint8_t* p, float (&z)[8], float& vmax) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&u.z);
    __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&u.w);
    const __nv_bfloat162 m = __hmax2_nan(__hmax2_nan(a, b), __hmax2_nan(c, d));
    vmax = fmax_nan(__low2float(m), __high2float(m));
    z[0] = __uint_as_float(u.x << 16);
    z[1] = __uint_as_float(u.x & 0xFFFF0000u);
    z[2] = __uint_as_float(u.y << 16);
    z[3] = __uint_as_float(u.y & 0xFFFF0000u);
    z[4] = __uint_as_float(u.z << 16);
    z[5] = __uint_as_float(u.z & 0xFFFF0000u);
    z[6] = __uint_as_float(u.w << 16);
    z[7] = __uint_as_float(u.w & 0xFFFF0000u);
  }
  static __device__ __forceinline__ float get(const uint8_t* tile, int j) {
    const uint16_t b = reinterpret_cast<const uint16_t*>(tile)[j];
    return __uint_as_float((uint32_t)b << 16);
  }
  static __device__ __forceinline__ float get_global(const void* row, int64_t j) {
    return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(row)[j] << 16);
  }
  static __device__ __forceinline__ void set_neg_inf(uint8_t* tile, int j) {
    reinterpret_cast<uint16_t*>(tile)[j] = 0xFF80u;
  }
};
template <>
struct VecT<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void load(const uint8_t* p, float (&z)[4], float& vmax) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    z[0] = u.x;
    z[1] = u.y;
    z[2] = u.z;
    z[3] = u.w;
    vmax = fmax_nan(fmax_nan(u.x, u.y), fmax_nan(u.z, u.w));
  }
  static __device__ __forceinline__ float get(const uint8_t* tile, int j) {
    return reinterpret_cast<const float*>(tile)[j];
  }
  static __device__ __forceinline__ float get_global(const void* row, int64_t j) {
    return reinterpret_cast<const float*>(row)[j];
  }
  static __device__ __forceinline__ void set_neg_inf(uint8_t* tile, int j) {
    reinterpret_cast<float*>(tile)[j] = -INFINITY;
  }
};

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

// Thread-private online softmax denominator.  Each element contributes 2^(z*c - R) with
// c = c_hi + c_lo = log2(e)/tau, evaluated as ex2(fma(z, c_lo, fma(z, c_hi, -R))) — two FFMAs and
// one MUFU.EX2, relative error ~2^-22.  R (binary32, exact) is rebased when an element would
// exceed 2^8 relative to it; the float64 accumulator is rescaled by an exact power difference.
struct LaneAcc {
  float R;     // exponent reference
  float thr;   // z above which a rebase is needed
  float mmax;  // exact max seen
  double acc;  // sum 2^(z*c - R)
  int bad;     // a NaN or +inf logit was seen
  __device__ __forceinline__ void reset() {
    R = -INFINITY;
    thr = -INFINITY;
    mmax = -INFINITY;
    acc = 0.0;
    bad = 0;
  }
};

// x * 2^d for an integer-valued d <= 0 (exact unless the result is subnormal)
__device__ __forceinline__ double scale_pow2(double x, float d) {
  if (!(d > -1022.0f)) return d > -2200.0f ? ldexp(x, (int)d) : 0.0;
  return x * __hiloint2double(((int)d + 1023) << 20, 0);
}

// The exponent reference R is an integer (floor(vmax * c_hi)), so every rescale of a sum by
// 2^(R_old - R_new) — here and in the partial reductions — is an exact power-of-two multiply.
__device__ __forceinline__ void lane_rebase(LaneAcc& a, float vmax, const RowCfg& rc) {
  const float Rn = floorf(vmax * rc.c_hi);
  if (a.acc != 0.0) a.acc = scale_pow2(a.acc, a.R - Rn);
  a.R = Rn;
  a.thr = (Rn + 8.0f) / rc.c_hi;
}

__device__ __forceinline__ float lane_exp(float z, const LaneAcc& a, const RowCfg& rc) {
  return ex2f(fmaf(z, rc.c_lo, fmaf(z, rc.c_hi, -a.R)));
}

// one scalar element into the accumulator (penalised entries)
__device__ __forceinline__ void lane_add(LaneAcc& a, float y, const RowCfg& rc) {
  if (y > -INFINITY) {
    if (y > a.thr) lane_rebase(a, y, rc);
    a.acc += (double)lane_exp(y, a, rc);
    a.mmax = fmaxf(a.mmax, y);
  }
}

}  // namespace smp

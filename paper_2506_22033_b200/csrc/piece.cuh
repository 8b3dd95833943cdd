// piece.cuh — geometry and encodings shared by the streaming kernel (phase A) and the per-row
// select kernel (phase B).
//
// Layout of the work (B200-first; the paper's CPU implementation walks a [B x V] column layout
// with per-row loops, P:364 — here the whole batch is one flattened stream):
//   * A row's local vocab slice is read as 16-byte vectors (8 bf16 / 4 f32).  Rows are padded
//     (virtually — nothing is read past the row) to Vq vectors, a multiple of one warp STEP
//     (128 vectors), and the padded [B x Vq] space is cut into equal spans, one per CTA.  A span
//     crossing a row boundary yields one "piece" per row.  Every boundary is STEP-aligned in row
//     coordinates, so a (step, lane) "group" — the 4 vectors lane l reads in step k, at row
//     vectors 128k + l + 32j — has the same index in the row whatever the CTA partition:
//     group id = 32k + l.
//   * The space is cut into equal STEP-aligned warp spans: every warp of phase A works alone (no
//     CTA barrier anywhere in phase A); a warp span crossing a row boundary yields one
//     "sub-piece" per row, and every sub-piece gets a warp record.
//   * Phase A writes, per group, the order-preserving bf16 key of the group max (rounded down)
//     to gkeys[row][group]; per sub-piece, a warp record with its max / exp-sum.
//   * Phase B: T = K-th largest key among the row's group keys and penalised elements.  K
//     distinct elements are >= val(T): T is a lower bound of the row's K-th largest z', and every
//     top-K element lies in a group whose key is >= T (or is penalised).  Only those groups are
//     re-read.
#pragma once
#include "common.cuh"
#include "elem.cuh"

namespace smp {

constexpr int kG = 4;                       // vectors per lane per step
constexpr int kStepVec = 32 * kG;           // vectors per warp step (= 4 groups of 32 lanes)
constexpr int kLaneList = 32;               // lane-max list entries per warp record
constexpr int kMaxRecW = 64;                // warp records per row (plan)

// warp record: RecHdr {m, flags, s, R = m * log2(e)/tau}
constexpr int kWarpRecBytes = kRecHdrBytes;
constexpr int kWarpRecStride = 64;
static_assert(kWarpRecBytes <= kWarpRecStride, "warp record layout");

__host__ __device__ inline int64_t vq_of(int vloc, int vec) {  // padded row length in vectors
  const int64_t nv = (vloc + vec - 1) / vec;
  return (nv + kStepVec - 1) / kStepVec * kStepVec;
}
__host__ __device__ inline int64_t groups_of(int64_t vq) { return vq / kG; }
// per-row key block in gkeys: [Vq / kG group keys | Vq / kStepVec step keys | pad to 8]
__host__ __device__ inline int64_t gk_stride(int64_t vq) { return (vq / kG + vq / kStepVec + 7) / 8 * 8; }

__device__ __forceinline__ uint4 ldg_stream(const uint8_t* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p));
  return u;
}

// order-preserving 16-bit key of a binary32 rounded DOWN to bf16 (exact for bf16 values);
// NaN maps to the +inf key (the row is flagged bad anyway)
__device__ __forceinline__ uint32_t key16_down(float f) {
  f = f + 0.0f;  // -0 -> +0
  uint32_t b = __float_as_uint(f);
  uint32_t h = b >> 16;
  if ((b >> 31) && (b & 0xFFFFu)) h += 1;  // negative with dropped bits: one bf16 step down
  if (h == 0xFF80u && f > -INFINITY) h = 0xFF7Fu;  // finite below the lowest bf16: its lowest finite key
  if (f != f) h = 0x7F80u;
  return h ^ ((h >> 15) ? 0xFFFFu : 0x8000u);
}
constexpr uint32_t kKey16NegInf = 0x007Fu;  // key16_down(-inf)
// the bf16 value of a 16-bit key (inverse of key16_down on bf16 values)
__device__ __forceinline__ float key16_val(uint32_t k) {
  const uint32_t h = k ^ ((k >> 15) ? 0x8000u : 0xFFFFu);
  return __uint_as_float(h << 16);
}

template <typename T>
struct Dec;
template <>
struct Dec<__nv_bfloat16> {
  static constexpr int N = 8;
  static constexpr uint32_t kNegInfWord = 0xFF80FF80u;
  static __device__ __forceinline__ float vmax(const uint4 u) {
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&u.z);
    __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&u.w);
    const __nv_bfloat162 m = __hmax2_nan(__hmax2_nan(a, b), __hmax2_nan(c, d));
    return fmax_nan(__low2float(m), __high2float(m));
  }
  static __device__ __forceinline__ float elem(const uint4 u, int i) {
    const uint32_t w = (i < 2) ? u.x : (i < 4) ? u.y : (i < 6) ? u.z : u.w;
    return __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
  }
  // elements whose bit is set in b (bit t = element t) become -inf
  static __device__ __forceinline__ uint4 mask(uint4 u, uint32_t b) {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if ((b >> (2 * i)) & 1u) w[i] = (w[i] & 0xFFFF0000u) | 0xFF80u;
      if ((b >> (2 * i + 1)) & 1u) w[i] = (w[i] & 0x0000FFFFu) | 0xFF800000u;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  static __device__ __forceinline__ float load1(const uint8_t* rowp, int i) {
    const unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(rowp) + i);
    return __uint_as_float((uint32_t)s << 16);
  }
};
template <>
struct Dec<float> {
  static constexpr int N = 4;
  static constexpr uint32_t kNegInfWord = 0xFF800000u;
  static __device__ __forceinline__ float vmax(const uint4 u) {
    return fmax_nan(fmax_nan(__uint_as_float(u.x), __uint_as_float(u.y)),
                    fmax_nan(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  static __device__ __forceinline__ float elem(const uint4 u, int i) {
    return __uint_as_float(i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w);
  }
  static __device__ __forceinline__ uint4 mask(uint4 u, uint32_t b) {
    if (b & 1u) u.x = kNegInfWord;
    if (b & 2u) u.y = kNegInfWord;
    if (b & 4u) u.z = kNegInfWord;
    if (b & 8u) u.w = kNegInfWord;
    return u;
  }
  static __device__ __forceinline__ float load1(const uint8_t* rowp, int i) {
    return __ldg(reinterpret_cast<const float*>(rowp) + i);
  }
};

// first index of the id-sorted entry list e[0..n) with id >= id0
__device__ __forceinline__ int uniq_lower_bound(const UniqEntry* e, int n, int id0) {
  int a = 0, b = n;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (e[mid].id < id0) a = mid + 1;
    else b = mid;
  }
  return a;
}

// bit t set <=> global id gid0 + t (t < VEC) is in the sorted list e[0..n)
template <int VEC>
__device__ __forceinline__ uint32_t listed_mask(const UniqEntry* e, int n, int gid0) {
  uint32_t m = 0;
  for (int i = uniq_lower_bound(e, n, gid0); i < n; ++i) {
    const int k = e[i].id - gid0;
    if (k >= VEC) break;
    m |= 1u << k;
  }
  return m;
}

}  // namespace smp

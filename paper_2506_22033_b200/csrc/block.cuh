// block.cuh — block-wide (CTA) primitives for 256-thread blocks: deterministic reductions, exact
// radix select of the K-th largest 64-bit composite and compaction in smem.
#pragma once
#include "common.cuh"

namespace smp {

constexpr int kBT = 256;            // consumer threads per CTA in the streaming / merge kernels
constexpr int kBW = kBT / 32;       // consumer warps

// Barrier among the kBT consumer threads only (named barrier 1), so that a warp-specialised
// producer warp outside [0, kBT) never has to join.
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kBT) : "memory"); }

struct BlockScratch {
  float* f;      // [kBW]
  double* d;     // [kBW]
  uint64_t* u;   // [kBW + 8]
  int* i;        // [kBW + 8]
};

// fixed-order (deterministic) float64 sum
__device__ __forceinline__ double block_sum_d(double v, const BlockScratch& s) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum_d(v);
  cbar();
  if (lane == 0) s.d[w] = v;
  cbar();
  double r = 0.0;
#pragma unroll
  for (int j = 0; j < kBW; ++j) r += s.d[j];
  return r;
}
__device__ __forceinline__ int block_sum_i(int v, const BlockScratch& s) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum_i(v);
  cbar();
  if (lane == 0) s.i[w] = v;
  cbar();
  int r = 0;
#pragma unroll
  for (int j = 0; j < kBW; ++j) r += s.i[j];
  return r;
}
__device__ __forceinline__ void block_minmax_u64(uint64_t mn, uint64_t mx, const BlockScratch& s, uint64_t* omn,
                                                 uint64_t* omx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  mn = warp_min_u64(mn);
  mx = warp_max_u64(mx);
  cbar();
  if (lane == 0) {
    s.u[w] = mn;
    reinterpret_cast<uint64_t*>(s.d)[w] = mx;
  }
  cbar();
  uint64_t a = s.u[0], b = reinterpret_cast<uint64_t*>(s.d)[0];
#pragma unroll
  for (int j = 1; j < kBW; ++j) {
    a = s.u[j] < a ? s.u[j] : a;
    const uint64_t t = reinterpret_cast<uint64_t*>(s.d)[j];
    b = t > b ? t : b;
  }
  *omn = a;
  *omx = b;
  cbar();
}

// Exact K-th largest among the NONZERO composites buf[0..n) (nonzero count > k >= 1, values
// unique).  Returns T with |{i : buf[i] >= T, buf[i] != 0}| == k.  8-bit digits, MSB first,
// starting at the first bit where the entries differ; early exit when a digit bin is taken whole.
__device__ __noinline__ uint64_t block_kth_largest(const uint64_t* buf, int n, int k, uint32_t* hist,
                                                   const BlockScratch& s) {
  uint64_t mn = ~0ull, mx = 0;
  for (int i = threadIdx.x; i < n; i += kBT) {
    const uint64_t c = buf[i];
    if (c) {
      mn = c < mn ? c : mn;
      mx = c > mx ? c : mx;
    }
  }
  block_minmax_u64(mn, mx, s, &mn, &mx);
  const int diff = (mn == mx) ? 0 : 64 - __clzll((long long)(mn ^ mx));  // bits that vary
  int d = ((diff + 7) / 8) * 8 - 8;                                    // top digit start
  if (d < 0) return mx;  // single distinct value (k == count)
  uint64_t prefix = mx >> (d + 8);  // common prefix above the first digit (d + 8 <= 64)
  if (d + 8 >= 64) prefix = 0;
  int need = k;
  for (; d >= 0; d -= 8) {
    for (int i = threadIdx.x; i < 256; i += kBT) hist[i] = 0;
    cbar();
    for (int i = threadIdx.x; i < n; i += kBT) {
      const uint64_t c = buf[i];
      if (c && ((d + 8 >= 64) || (c >> (d + 8)) == prefix)) atomicAdd(&hist[(uint32_t)(c >> d) & 255u], 1u);
    }
    cbar();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t c8[8];
      int ls = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c8[j] = hist[255 - 8 * lane - j];
        ls += (int)c8[j];
      }
      const int incl = warp_incl_scan_i(ls, lane);
      const int excl = incl - ls;
      if (excl < need && need <= incl) {
        int acc = excl;
        for (int j = 0; j < 8; ++j) {
          if (acc + (int)c8[j] >= need) {
            s.i[kBW + 0] = 255 - 8 * lane - j;
            s.i[kBW + 1] = acc;
            s.i[kBW + 2] = (int)c8[j];
            break;
          }
          acc += (int)c8[j];
        }
      }
    }
    cbar();
    const int digit = s.i[kBW + 0], above = s.i[kBW + 1], bincnt = s.i[kBW + 2];
    cbar();
    prefix = (prefix << 8) | (uint64_t)digit;
    need -= above;
    if (bincnt == need) return prefix << d;
  }
  return prefix;
}

// Keep the nonzero entries >= T (order not preserved).  Returns the new count; *kmin = min kept.
// Uses `tmp` (>= n entries of scratch) to stage.
__device__ __forceinline__ int block_compact_ge(uint64_t* buf, int n, uint64_t T, int* counter,
                                                const BlockScratch& s, uint64_t* kmin) {
  constexpr int kMaxPer = 12;  // n <= kBT * kMaxPer (3072 = the candidate area)
  uint64_t v[kMaxPer];
  uint64_t mn = ~0ull;
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j) {
    const int i = threadIdx.x + j * kBT;
    v[j] = (i < n) ? buf[i] : 0;
  }
  if (threadIdx.x == 0) *counter = 0;
  cbar();
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j) {
    if (v[j] && v[j] >= T) {
      buf[atomicAdd(counter, 1)] = v[j];
      mn = v[j] < mn ? v[j] : mn;
    }
  }
  cbar();
  const int out = *counter;
  uint64_t a, b;
  block_minmax_u64(mn, 0, s, &a, &b);
  *kmin = a;
  return out;
}

}  // namespace smp

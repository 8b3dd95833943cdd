// warp_cand.cuh — per-warp top-K candidate buffer with a running admission threshold.
//
// Top-k ("restrict candidates") without a full sort: every warp keeps
// the exact top-K composites (z' desc, id asc) of what it has streamed in a shared-memory
// buffer.  Elements below the running threshold theta (= value of the current K-th best) are
// rejected with one compare per 16-byte vector; survivors are appended with a ballot/popc
// prefix; when the buffer passes half full it is shrunk back to K entries with a warp radix
// select on the 64-bit composite (8-bit digits, MSB first, early exit).  Exact: an element is
// only ever dropped when K better composites are known.
#pragma once
#include "common.cuh"

namespace smp {

constexpr int kCapW = 512;            // buffer entries per warp
constexpr int kShrinkAt = kCapW - 256; // after a push, shrink if cnt exceeds this

struct WarpCand {
  uint64_t* buf;    // smem [kCapW]
  uint32_t* hist;   // smem [256]
  int cnt;          // warp-uniform
  int keff;         // K kept per shrink
  float theta;      // admission threshold on z' (warp-uniform)
  bool dropped;     // some element was rejected / dropped (the list is not the whole range)

  __device__ void reset(int k) {
    cnt = 0;
    keff = k;
    theta = -3.402823466e38f;  // admits every finite value, rejects -inf
    dropped = false;
  }
};

// Exact K-th largest of buf[0..n) (n > k >= 1, composites unique); returns T with
// |{i : buf[i] >= T}| == k.
__device__ __noinline__ uint64_t warp_kth_largest(const uint64_t* buf, int n, int k, uint32_t* hist,
                                                  int lane) {
  uint64_t prefix = 0;  // digits chosen so far (right-aligned)
  int need = k;
  for (int d = 56; d >= 0; d -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const uint64_t c = buf[i];
      const bool match = (d == 56) ? true : ((c >> (d + 8)) == prefix);
      if (match) atomicAdd(&hist[(uint32_t)(c >> d) & 255u], 1u);
    }
    __syncwarp();
    // lane L owns bins [255-8L-7, 255-8L]; scan from the top bin down.
    uint32_t cnt8[8];
    uint32_t lsum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      cnt8[j] = hist[255 - 8 * lane - j];
      lsum += cnt8[j];
    }
    const int incl = warp_incl_scan_i((int)lsum, lane);
    const int excl = incl - (int)lsum;
    const bool mine = (excl < need) && (need <= incl);
    const unsigned who = __ballot_sync(kFull, mine);
    const int src = __ffs(who) - 1;
    int digit = 0, above = 0, bincnt = 0;
    if (lane == src) {
      int acc = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (acc + (int)cnt8[j] >= need) {
          digit = 255 - 8 * lane - j;
          above = acc;
          bincnt = (int)cnt8[j];
          break;
        }
        acc += (int)cnt8[j];
      }
    }
    digit = __shfl_sync(kFull, digit, src);
    above = __shfl_sync(kFull, above, src);
    bincnt = __shfl_sync(kFull, bincnt, src);
    __syncwarp();
    prefix = (prefix << 8) | (uint64_t)digit;
    need -= above;
    if (bincnt == need) return prefix << d;  // every element of this bin is selected
  }
  return prefix;  // exact composite of the K-th
}

// Keep exactly the entries >= T (in place, order preserved).  Returns the new count and
// the minimum kept composite in *kmin.
__device__ __forceinline__ int warp_compact_ge(uint64_t* buf, int n, uint64_t T, int lane,
                                               uint64_t* kmin) {
  int out = 0;
  uint64_t mn = ~0ull;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    uint64_t c = 0;
    bool keep = false;
    if (i < n) {
      c = buf[i];
      keep = c >= T;
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    __syncwarp();
    if (keep) {
      buf[out + __popc(bal & ((1u << lane) - 1u))] = c;
      mn = c < mn ? c : mn;
    }
    out += __popc(bal);
    __syncwarp();
  }
  *kmin = warp_min_u64(mn);
  return out;
}

__device__ __forceinline__ void warp_shrink(WarpCand& w, int lane) {
  if (w.cnt <= w.keff) return;
  const uint64_t T = warp_kth_largest(w.buf, w.cnt, w.keff, w.hist, lane);
  uint64_t kmin;
  w.cnt = warp_compact_ge(w.buf, w.cnt, T, lane, &kmin);
  w.theta = comp_val(kmin);
  w.dropped = true;
}

// Two-phase append: every lane calls warp_push_slot(np) to get its first slot, writes its np
// composites to buf[slot..slot+np), then all lanes call warp_push_done(total).
__device__ __forceinline__ int warp_push_slot(const WarpCand& w, int np, int lane, int* total) {
  const int incl = warp_incl_scan_i(np, lane);
  *total = __shfl_sync(kFull, incl, 31);
  return w.cnt + incl - np;
}
__device__ __forceinline__ void warp_push_done(WarpCand& w, int total, int lane) {
  w.cnt += total;
  __syncwarp();
  if (w.cnt > kShrinkAt) warp_shrink(w, lane);
}

// Append this lane's `np` composites (vals[0..np)) to the warp buffer.
template <int NV>
__device__ __forceinline__ void warp_push(WarpCand& w, const uint64_t (&vals)[NV], int np, int lane) {
  const int incl = warp_incl_scan_i(np, lane);
  const int total = __shfl_sync(kFull, incl, 31);
  int pos = w.cnt + incl - np;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (j < np) w.buf[pos + j] = vals[j];
  w.cnt += total;
  __syncwarp();
  if (w.cnt > kShrinkAt) warp_shrink(w, lane);
}

// Bitonic sort of buf[0..n) descending (n <= npow2 <= kCapW); pads with 0 (sorts last).
__device__ __forceinline__ void warp_sort_desc(uint64_t* buf, int n, int lane) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + lane; i < N; i += 32) buf[i] = 0;
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < N; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = buf[i], b = buf[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Bitonic sort ascending of buf[0..n).
__device__ __forceinline__ void warp_sort_asc(uint64_t* buf, int n, int lane) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + lane; i < N; i += 32) buf[i] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < N; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = buf[i], b = buf[ixj];
          const bool asc = (i & k) == 0;
          if (asc ? (a > b) : (a < b)) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace smp

// stream.cuh — phase A of the sampling step: logits [B x V] -> per-piece partial records.
//
// Work decomposition (B200-first; not the paper's CPU column layout):
//   The padded logits space [B x Vp] is flattened and cut into equal contiguous spans (<= 16384
//   16-byte vectors each), one per CTA, 3 CTAs per SM (exact load balance at any B — no
//   1.73-rows-per-SM wave quantisation at B=256).  A span that crosses a row boundary yields one
//   "piece" per row.  Within a piece every warp streams its own contiguous eighth with 16-byte
//   read-only global loads, G = 4 vectors (32 logits) per lane per step, the next step's loads
//   issued before the current step is computed; warps never wait for each other.
//
//   Pass 1 (the hot loop, no data-dependent work): per 16-byte vector one NaN-propagating max,
//   the exp-sum (2 FFMA + 1 MUFU.EX2 per logit into a float64 accumulator) and one 2-byte store
//   of the vector max (order-preserving bf16 key, rounded down) into shared memory.  Steps that
//   hold a penalised id or the row's padding tail take an out-of-line path (penalties applied as
//   a sparse scatter from the slot's incremental unique-token table).
//   Pass 2 (per piece, from shared memory + L2): T = the K-th largest vector max, found by binary
//   search on the keys — K distinct elements are >= T, so T is a lower bound of the piece's K-th
//   largest element and every top-K element lies in a vector whose max is >= T.  Only those few
//   vectors are re-read (from L2) to collect the exact candidates, which are reduced to the exact
//   top-K (radix select), sorted, and written with the piece's max / exp-sum to the record.
//   Phase B (merge_rows_kernel, one CTA per row) combines a row's records into the sample.
#pragma once
#include "block.cuh"
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"

namespace smp {

constexpr int kG = 4;              // 16-byte vectors per lane per step
constexpr int kMaxSpanVec = 12288; // vectors per CTA span (vector-max keys live in smem)
constexpr int kCapW = 384;         // warp candidate region entries (pass 2)
constexpr int kCap = kBW * kCapW;  // candidate area
constexpr int kPenWin = 1024;      // penalty entries staged in smem per piece
constexpr int kQW = 256;          // warp list of qualifying vector indices (pass 2)
constexpr int kCtasPerSm = 3;

// pass-2 per-warp partial (smem)
struct WarpPart {
  float m;
  int bad;
  double s;
  double R;
  int cnt;
  int pad;
  uint64_t floor;
};

// shared-memory carve-up (phase A)
constexpr int kOffVkey = 0;                                   // [kMaxSpanVec] u16
constexpr int kOffCand = kOffVkey + kMaxSpanVec * 2;          // [kCap] u64
constexpr int kOffPen = kOffCand + kCap * 8;                  // [kPenWin] UniqEntry
constexpr int kOffHist = kOffPen + kPenWin * 8;               // [kBW][256] u32 (warp hists; [0] CTA)
constexpr int kOffQl = kOffHist + kBW * 256 * 4;             // [kBW][kQW] u32
constexpr int kOffScr = kOffQl + kBW * kQW * 4;               // f[8] d[8] u[16] i[16]
constexpr int kOffCtl = kOffScr + 288;                        // ints [32]
constexpr int kOffParts = kOffCtl + 128;                      // [kBW] WarpPart
constexpr int kStreamSmem = kOffParts + kBW * (int)sizeof(WarpPart);
static_assert(kStreamSmem * kCtasPerSm <= 227 * 1024, "phase-A smem exceeds the SM budget");
static_assert(kMaxSpanVec % 8 == 0, "vector keys are scanned 8 per 16-byte word");

struct StreamArgs {
  const void* logits;
  int64_t ld;          // row stride (elements)
  int B;
  int V;               // global vocab
  int voff, vloc;      // local slice
  int Vp;              // vloc rounded up to the vector width
  int64_t span;        // elements per CTA (multiple of the vector width)
  int64_t N;           // B * Vp
  const int32_t* slots;
  const sampling_params* params_dev;  // nullable
  const sampling_params* params_tab;
  int kcand;
  int pen_mode;
  HistState hs;
  uint8_t* records;
  int64_t rec_stride;
  uint64_t* trace;     // debug: per-CTA phase timestamps (globaltimer ns), nullable
};

#define TRACE(k)                                                                   \
  do {                                                                             \
    if (a.trace) cbar(); /* CTA-level phase boundary (debug only) */               \
    if (a.trace && threadIdx.x == 0) {                                             \
      uint64_t t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
      a.trace[(int64_t)blockIdx.x * 32 + (k)] = t_;                                \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint8_t* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p));
  return u;
}

// order-preserving 16-bit key of a binary32 rounded DOWN to bf16 (exact for bf16 values)
__device__ __forceinline__ uint32_t key16_down(float f) {
  f = f + 0.0f;  // -0 -> +0
  uint32_t b = __float_as_uint(f);
  uint32_t h = b >> 16;
  if ((b >> 31) && (b & 0xFFFFu)) h += 1;  // negative with dropped bits: one bf16 step down
  if (f != f) h = 0x7F80u;                 // NaN (row is flagged bad anyway): treat as +inf
  return h ^ ((h >> 15) ? 0xFFFFu : 0x8000u);
}
__device__ __forceinline__ float key16_to_f(uint32_t k) {
  const uint32_t h = k ^ ((k >> 15) ? 0x8000u : 0xFFFFu);
  return __uint_as_float((h & 0xFFFFu) << 16);
}

// Exact K-th largest of buf[0..n) (n > k >= 1, unique composites) by one warp; returns T with
// exactly k entries >= T.  8-bit digits from the first differing bit; early exit.
__device__ __noinline__ uint64_t warp_kth_largest(const uint64_t* buf, int n, int k, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t mn = ~0ull, mx = 0;
  for (int i = lane; i < n; i += 32) {
    const uint64_t c = buf[i];
    mn = c < mn ? c : mn;
    mx = c > mx ? c : mx;
  }
  mn = warp_min_u64(mn);
  mx = warp_max_u64(mx);
  const int diff = (mn == mx) ? 0 : 64 - __clzll((long long)(mn ^ mx));
  int d = ((diff + 7) / 8) * 8 - 8;
  if (d < 0) return mx;
  uint64_t prefix = (d + 8 >= 64) ? 0 : (mx >> (d + 8));
  int need = k;
  for (; d >= 0; d -= 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hist[lane * 8 + j] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const uint64_t c = buf[i];
      if ((d + 8 >= 64) || (c >> (d + 8)) == prefix) atomicAdd(&hist[(uint32_t)(c >> d) & 255u], 1u);
    }
    __syncwarp();
    uint32_t c8[8];
    int ls = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c8[j] = hist[255 - 8 * lane - j];
      ls += (int)c8[j];
    }
    const int incl = warp_incl_scan_i(ls, lane);
    const int excl = incl - ls;
    const unsigned who = __ballot_sync(kFull, excl < need && need <= incl);
    const int src = __ffs(who) - 1;
    int digit = 0, above = 0, bincnt = 0;
    if (lane == src) {
      int acc = excl;
      for (int j = 0; j < 8; ++j) {
        if (acc + (int)c8[j] >= need) {
          digit = 255 - 8 * lane - j;
          above = acc;
          bincnt = (int)c8[j];
          break;
        }
        acc += (int)c8[j];
      }
    }
    digit = __shfl_sync(kFull, digit, src);
    above = __shfl_sync(kFull, above, src);
    bincnt = __shfl_sync(kFull, bincnt, src);
    __syncwarp();
    prefix = (prefix << 8) | (uint64_t)digit;
    need -= above;
    if (bincnt == need) return prefix << d;
  }
  return prefix;
}

// Bitonic sort of one value per lane, descending across the warp (lane 0 = largest).
__device__ __forceinline__ uint32_t warp_sort_desc_u32(uint32_t x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(kFull, x, j);
      const bool desc = (lane & k) == 0;  // k == 32: the whole warp descending
      const bool lower = (lane & j) == 0;
      x = (lower == desc) ? max(x, y) : min(x, y);
    }
  return x;
}

// Keep buf[i] >= T of buf[0..n) in place (order preserved); returns the new count.
__device__ __forceinline__ int warp_compact_ge(uint64_t* buf, int n, uint64_t T) {
  const int lane = threadIdx.x & 31;
  int out = 0;
  for (int b0 = 0; b0 < n; b0 += 32) {
    const int i = b0 + lane;
    const uint64_t c = (i < n) ? buf[i] : 0;
    const bool keep = i < n && c >= T;
    const unsigned bal = __ballot_sync(kFull, keep);
    __syncwarp();
    if (keep) buf[out + __popc(bal & ((1u << lane) - 1u))] = c;
    out += __popc(bal);
    __syncwarp();
  }
  return out;
}

// Bitonic sort of buf[0..n) descending by one warp (buf has room for the next power of two).
__device__ __forceinline__ void warp_sort_desc(uint64_t* buf, int n) {
  const int lane = threadIdx.x & 31;
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + lane; i < N; i += 32) buf[i] = 0;
  __syncwarp();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < N; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = buf[i], y = buf[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (x < y) : (x > y)) {
            buf[i] = y;
            buf[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
}

template <typename T>
struct Dec;
template <>
struct Dec<__nv_bfloat16> {
  static __device__ __forceinline__ void run(const uint4 u, float (&z)[8], float& vmax) {
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
  static constexpr uint32_t kNegInfWord = 0xFF80FF80u;
};
template <>
struct Dec<float> {
  static __device__ __forceinline__ void run(const uint4 u, float (&z)[4], float& vmax) {
    z[0] = __uint_as_float(u.x);
    z[1] = __uint_as_float(u.y);
    z[2] = __uint_as_float(u.z);
    z[3] = __uint_as_float(u.w);
    vmax = fmax_nan(fmax_nan(z[0], z[1]), fmax_nan(z[2], z[3]));
  }
  static __device__ __forceinline__ float vmax(const uint4 u) {
    return fmax_nan(fmax_nan(__uint_as_float(u.x), __uint_as_float(u.y)),
                    fmax_nan(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  static __device__ __forceinline__ float elem(const uint4 u, int i) {
    return __uint_as_float(i == 0 ? u.x : i == 1 ? u.y : i == 2 ? u.z : u.w);
  }
  static constexpr uint32_t kNegInfWord = 0xFF800000u;
};

// Piece context handed to the out-of-line paths (by value: no register array escapes).
struct PieceCtx {
  const uint8_t* rowp;    // first byte of the piece
  const UniqEntry* psrc;  // the piece's penalty entries (sorted ids)
  int pcount;
  int gid0;               // global id of the piece's first element
  int lid_end;            // piece-relative ids >= lid_end are padding
  int pen_mode;
};

// first entry with piece-relative id >= lo (binary search over the sorted list)
__device__ __forceinline__ int entry_lower_bound(const PieceCtx& pc, int lo) {
  int a = 0, b = pc.pcount;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (pc.psrc[mid].id - pc.gid0 < lo) a = mid + 1;
    else b = mid;
  }
  return a;
}

// Apply every override to the decoded vector v: penalised entries (OPENAI_CTRL / LINEAR)
// and the padding tail (-inf).
template <int VEC>
__device__ __forceinline__ void apply_overrides(const PieceCtx& pc, int v, const sampling_params& prm,
                                                float (&z)[VEC], int& bad) {
  if (pc.pcount > 0)
    for (int e = entry_lower_bound(pc, v * VEC); e < pc.pcount; ++e) {
      const UniqEntry ue = pc.psrc[e];
      const int k = ue.id - pc.gid0 - v * VEC;
      if (k >= VEC) break;
#pragma unroll
      for (int t = 0; t < VEC; ++t)
        if (t == k) {
          bad |= !(z[t] < INFINITY) ? 1 : 0;
          z[t] = apply_penalty(z[t], ue.meta, prm, pc.pen_mode);
        }
    }
#pragma unroll
  for (int t = 0; t < VEC; ++t)
    if (v * VEC + t >= pc.lid_end) z[t] = -INFINITY;
}

// A step holding a penalised id or the padding tail (out-of-line; re-reads the step from L2).
template <typename T>
__device__ __noinline__ LaneAcc slow_step(PieceCtx pc, LaneAcc la, int vb, int wv1, uint16_t* vkey,
                                          const sampling_params* sprm, RowCfg rc) {
  const sampling_params prm = *sprm;
  constexpr int VEC = VecT<T>::N;
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < kG; ++j) {
    const int v = vb + lane + 32 * j;
    if (v >= wv1) continue;
    float z[VEC], vm0;
    Dec<T>::run(ldg_stream(pc.rowp + (int64_t)v * 16), z, vm0);
    apply_overrides<VEC>(pc, v, prm, z, la.bad);
    float vm = -INFINITY;
#pragma unroll
    for (int t = 0; t < VEC; ++t) vm = fmax_nan(vm, z[t]);
    la.bad |= !(vm < INFINITY) ? 1 : 0;
    if (vm > -INFINITY) {
      if (vm > la.thr) lane_rebase(la, vm, rc);
      float s = 0.f;
#pragma unroll
      for (int t = 0; t < VEC; ++t) s += lane_exp(z[t], la, rc);
      la.acc += (double)s;
      la.mmax = fmaxf(la.mmax, vm);
    }
    vkey[v] = (uint16_t)key16_down(vm);
  }
  return la;
}

template <typename T>
__global__ void __launch_bounds__(kBT, kCtasPerSm) stream_kernel(const StreamArgs a) {
  constexpr int VEC = VecT<T>::N;
  constexpr int ESZ = (int)sizeof(T);
  constexpr int STEP = 32 * kG;  // vectors per warp step

  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint4 kNegInfVec = make_uint4(Dec<T>::kNegInfWord, Dec<T>::kNegInfWord, Dec<T>::kNegInfWord,
                                      Dec<T>::kNegInfWord);
  const int64_t a0 = (int64_t)blockIdx.x * a.span;
  const int64_t a1 = min(a.N, a0 + a.span);
  if (a0 >= a1) return;
  TRACE(0);

  uint16_t* vkey = reinterpret_cast<uint16_t*>(smem + kOffVkey);
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem + kOffCand);
  UniqEntry* pen = reinterpret_cast<UniqEntry*>(smem + kOffPen);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + kOffHist);
  uint32_t* whist = hist + wid * 256;
  BlockScratch bs;
  bs.f = reinterpret_cast<float*>(smem + kOffScr);
  bs.d = reinterpret_cast<double*>(smem + kOffScr + 32);
  bs.u = reinterpret_cast<uint64_t*>(smem + kOffScr + 96);
  bs.i = reinterpret_cast<int*>(smem + kOffScr + 224);
  int* ctl = reinterpret_cast<int*>(smem + kOffCtl);  // [2] CTA bound key, [6..7] K-th composite
  uint32_t* qlist = reinterpret_cast<uint32_t*>(smem + kOffQl);
  WarpPart* parts = reinterpret_cast<WarpPart*>(smem + kOffParts);
  uint32_t* tkey = reinterpret_cast<uint32_t*>(&ctl[2]);
  sampling_params* sprm = reinterpret_cast<sampling_params*>(&ctl[16]);  // the piece row's params
  if (tid == 0) *tkey = 0;
  const uint8_t* lg = reinterpret_cast<const uint8_t*>(a.logits);
  int ntr = 1;

  int64_t pos = a0;
  while (pos < a1) {
    // ---------------- piece = [pos, pend) of row r
    const int r = (int)(pos / a.Vp);
    const int loc0 = (int)(pos - (int64_t)r * a.Vp);
    const int64_t pend = min(a1, (int64_t)(r + 1) * a.Vp);
    const int plen = (int)(pend - pos);
    PieceCtx pc;
    pc.rowp = lg + ((int64_t)r * a.ld + loc0) * ESZ;
    const int nv = plen / VEC;
    const int per = ((nv + kBW - 1) / kBW + 7) & ~7;  // warp key ranges 16-byte aligned
    const int wv0 = min(nv, wid * per);
    const int wv1 = min(nv, wv0 + per);
    pc.gid0 = a.voff + loc0;
    pc.lid_end = a.vloc - loc0;
    pc.pen_mode = a.pen_mode;
    // first loads go out before any metadata round trip
    uint4 u[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int v = wv0 + lane + 32 * j;
      u[j] = (v < wv1) ? ldg_stream(pc.rowp + (int64_t)v * 16) : kNegInfVec;
    }
    const int slot = a.slots ? a.slots[r] : r;
    const sampling_params* gprm = a.params_dev ? a.params_dev + r : a.params_tab + slot;
    const RowCfg rc = decode_row(*gprm, a.V, a.kcand);
    if (tid == 0) *sprm = *gprm;
    // penalty entries with global ids in [gid0, g1)
    const UniqEntry* utab = a.hs.uniq + (int64_t)slot * a.hs.L;
    const int nu = a.hs.meta[slot].n_uniq;
    const int g1 = a.voff + min(a.vloc, loc0 + plen);
    int lo = 0, hi = 0;
    for (int i = tid; i < nu; i += kBT) {
      const int id = utab[i].id;
      lo += id < pc.gid0;
      hi += id < g1;
    }
    if (tid < 8 && nv + tid < ((nv + 7) & ~7)) vkey[nv + tid] = 0;  // key words past the piece
    lo = block_sum_i(lo, bs);
    hi = block_sum_i(hi, bs);
    pc.pcount = hi - lo;
    pc.psrc = (pc.pcount <= kPenWin) ? pen : utab + lo;  // smem copy unless huge
    if (pc.pcount <= kPenWin)
      for (int i = tid; i < pc.pcount; i += kBT) pen[i] = utab[lo + i];
    cbar();
    TRACE(ntr++);
    LaneAcc la;
    la.reset();
    // this warp's first penalty entry
    int wcur = entry_lower_bound(pc, wv0 * VEC);
    int next_pen = (wcur < pc.pcount) ? pc.psrc[wcur].id - pc.gid0 : 0x7FFFFFFF;

    // ================= pass 1: stream =================
    for (int vb = wv0; vb < wv1; vb += STEP) {
      const int s1 = min(wv1, vb + STEP) * VEC;  // piece-relative end of this step
      if (next_pen < s1 || s1 > pc.lid_end) {    // rare: penalised ids / padding in this step
        la = slow_step<T>(pc, la, vb, wv1, vkey, sprm, rc);
        wcur = entry_lower_bound(pc, s1);
        next_pen = (wcur < pc.pcount) ? pc.psrc[wcur].id - pc.gid0 : 0x7FFFFFFF;
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          const int v = vb + STEP + lane + 32 * j;
          u[j] = (v < wv1) ? ldg_stream(pc.rowp + (int64_t)v * 16) : kNegInfVec;
        }
        continue;
      }
      uint4 cur[kG];  // this step's vectors (lanes past the warp's range hold -inf)
      float vm[kG];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        cur[j] = u[j];
        vm[j] = Dec<T>::vmax(cur[j]);
      }
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int v = vb + STEP + lane + 32 * j;
        u[j] = (v < wv1) ? ldg_stream(pc.rowp + (int64_t)v * 16) : kNegInfVec;
      }
      float gmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        la.bad |= !(vm[j] < INFINITY) ? 1 : 0;
        gmax = fmaxf(gmax, vm[j]);
        if (vb + lane + 32 * j < wv1) vkey[vb + lane + 32 * j] = (uint16_t)key16_down(vm[j]);
      }
      if (gmax > -INFINITY) {
        if (gmax > la.thr) lane_rebase(la, gmax, rc);
        float sj[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          float e[VEC];
#pragma unroll
          for (int i = 0; i < VEC; ++i) e[i] = lane_exp(Dec<T>::elem(cur[j], i), la, rc);
#pragma unroll
          for (int st = 1; st < VEC; st <<= 1)
#pragma unroll
            for (int i = 0; i < VEC; i += 2 * st) e[i] += e[i + st];
          sj[j] = e[0];
        }
        la.acc += (double)((sj[0] + sj[1]) + (sj[2] + sj[3]));
        la.mmax = fmaxf(la.mmax, gmax);
      }
    }
    TRACE(ntr++);
    cbar();  // all vector keys of the piece are in smem

    // ================= pass 2: bound, collect, top-K =================
    // (1) bound: T = the K-th largest of the 256 lane maxima (each lane's max over the vectors it
    //     streamed).  K distinct lanes, hence K distinct elements, are >= T, so T is a lower bound
    //     of the piece's K-th largest element.  Per-warp shuffle sort, then every lane counts the
    //     entries >= its own value in all 8 sorted lists (8 independent 5-step searches).
    const int keff = rc.keff;
    const sampling_params prm = *sprm;
    {
      uint32_t x = (la.mmax > -INFINITY) ? f2key(la.mmax) : 0u;  // 0 = no finite element
      x = warp_sort_desc_u32(x, lane);
      uint32_t* lists = hist;  // [kBW][32] descending
      lists[wid * 32 + lane] = x;
      cbar();
      if (x != 0) {
        int pos[kBW];
#pragma unroll
        for (int w = 0; w < kBW; ++w) pos[w] = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1)
#pragma unroll
          for (int w = 0; w < kBW; ++w) pos[w] += (lists[w * 32 + pos[w] + st - 1] >= x) ? st : 0;
        int c = 0;
#pragma unroll
        for (int w = 0; w < kBW; ++w) c += pos[w] + ((pos[w] == 31 && lists[w * 32 + 31] >= x) ? 1 : 0);
        if (c >= keff) atomicMax(tkey, x);
      }
      cbar();
    }
    TRACE(ntr++);
    const uint32_t kNegInf = key16_down(-INFINITY);
    const bool bounded = *tkey != 0u;
    const float Tv = bounded ? key2f(*tkey) : -3.402823466e38f;
    // vectors that can hold an element >= T (unbounded: every vector with a finite element)
    const uint32_t lo_k = bounded ? max(key16_down(Tv), kNegInf + 1) : kNegInf + 1;
    // (2) collect: the qualifying vectors of this warp (key >= lo_k) are listed first (smem only),
    //     then re-read from L2 in batches of 4 per lane (one round trip per batch), exact values
    //     (penalties / padding re-applied), every element >= T appended to the warp region
    uint64_t* wreg = cand + wid * kCapW;
    uint32_t* ql = qlist + wid * kQW;
    int wc = 0;
    uint64_t wfloor = 0;  // composites < wfloor were dropped by a warp shrink
    const uint4* wk4 = reinterpret_cast<const uint4*>(vkey + wv0);
    const int n4 = (wv1 - wv0 + 7) >> 3;
    const uint32_t lo2 = lo_k | (lo_k << 16);
    for (int p4 = 0; p4 < n4;) {
      int nq = 0;
      while (p4 < n4) {  // 8 keys per lane per round; words past the piece hold key 0 < lo_k
        uint32_t bits = 0;
        if (p4 + lane < n4) {
          const uint4 q = wk4[p4 + lane];
          const uint32_t w4[4] = {__vcmpgeu2(q.x, lo2), __vcmpgeu2(q.y, lo2), __vcmpgeu2(q.z, lo2),
                                  __vcmpgeu2(q.w, lo2)};
#pragma unroll
          for (int t = 0; t < 4; ++t) bits |= ((w4[t] & 1u) | ((w4[t] >> 30) & 2u)) << (2 * t);
        }
        const int c = __popc(bits);
        const int incl = warp_incl_scan_i(c, lane);
        const int tot_r = __shfl_sync(kFull, incl, 31);
        if (nq + tot_r > kQW) break;  // list full: process it first (a round adds <= 256 = kQW)
        int off = nq + incl - c;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          ql[off++] = (uint32_t)(wv0 + (p4 + lane) * 8 + b);
        }
        nq += tot_r;
        p4 += 32;
      }
      __syncwarp();
      for (int b0 = 0; b0 < nq; b0 += 32 * kG) {
        uint4 ld[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          const int i = b0 + lane + 32 * j;
          if (i < nq) ld[j] = ldg_stream(pc.rowp + (int64_t)ql[i] * 16);
        }
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          const int i = b0 + lane + 32 * j;
          if (!__any_sync(kFull, i < nq)) break;
          float z[VEC];
          int v = 0;
          uint32_t msk = 0;
          if (i < nq) {
            v = (int)ql[i];
            float vm;
            Dec<T>::run(ld[j], z, vm);
            int bad_unused = 0;
            apply_overrides<VEC>(pc, v, prm, z, bad_unused);
#pragma unroll
            for (int t = 0; t < VEC; ++t)
              msk |= (z[t] >= Tv && z[t] > -INFINITY && z[t] < INFINITY &&
                      make_comp(z[t], pc.gid0 + v * VEC + t) >= wfloor) ? (1u << t) : 0u;
          }
          int total = warp_sum_i(__popc(msk));
          if (wc + total > kCapW) {  // rare: keep the warp's exact top-K, raise the floor
            const uint64_t Tc = warp_kth_largest(wreg, wc, keff, whist);
            wc = warp_compact_ge(wreg, wc, Tc);
            wfloor = Tc > wfloor ? Tc : wfloor;
#pragma unroll
            for (int t = 0; t < VEC; ++t)
              if (((msk >> t) & 1u) && make_comp(z[t], pc.gid0 + v * VEC + t) < wfloor) msk &= ~(1u << t);
            total = warp_sum_i(__popc(msk));
          }
          const int n_l = __popc(msk);
          int pos = wc + warp_incl_scan_i(n_l, lane) - n_l;
#pragma unroll
          for (int t = 0; t < VEC; ++t)
            if ((msk >> t) & 1u) wreg[pos++] = make_comp(z[t], pc.gid0 + v * VEC + t);
          wc += total;
          __syncwarp();
        }
      }
    }
    TRACE(ntr++);
    // (3) warp: exact top-K of its candidates, sorted; partial reductions
    if (wc > keff) {
      const uint64_t Tc = warp_kth_largest(wreg, wc, keff, whist);
      wc = warp_compact_ge(wreg, wc, Tc);
      wfloor = Tc > wfloor ? Tc : wfloor;
    }
    warp_sort_desc(wreg, wc);
    {
      const float m = warp_max(la.mmax);
      float Rl = la.acc != 0.0 ? la.R : -INFINITY;
      Rl = warp_max(Rl);
      double sv = (la.acc != 0.0) ? la.acc * exp2((double)la.R - (double)Rl) : 0.0;
      sv = warp_sum_d(sv);
      const int bad = __any_sync(kFull, la.bad);
      if (lane == 0) {
        WarpPart wp;
        wp.m = m;
        wp.bad = bad;
        wp.s = sv;
        wp.R = (double)Rl;
        wp.cnt = wc;
        wp.pad = 0;
        wp.floor = wfloor;
        parts[wid] = wp;
      }
    }
    cbar();
    TRACE(ntr++);
    // (4) CTA: rank-merge the 8 sorted lists (binary search per list) straight into the record
    int offs[kBW + 1];
    offs[0] = 0;
#pragma unroll
    for (int w = 0; w < kBW; ++w) offs[w + 1] = offs[w] + parts[w].cnt;
    const int tot = offs[kBW];
    const int n = tot < keff ? tot : keff;
    uint8_t* rec = a.records + ((int64_t)blockIdx.x + r) * a.rec_stride;
    uint64_t* ent = reinterpret_cast<uint64_t*>(rec + kRecHdrBytes);
    for (int e = tid; e < tot; e += kBT) {
      int w = 0;
#pragma unroll
      for (int q = 1; q < kBW; ++q) w += (e >= offs[q]);
      const int qi = e - offs[w];
      const uint64_t c = cand[w * kCapW + qi];
      // rank = entries greater than c in all lists (own list: its index); the 8 searches
      // (binary lifting over <= 128 sorted entries) run side by side
      int pos[kBW], lim[kBW];
#pragma unroll
      for (int o = 0; o < kBW; ++o) {
        pos[o] = 0;
        lim[o] = (o == w) ? 0 : parts[o].cnt;
      }
#pragma unroll
      for (int st = 128; st; st >>= 1)
#pragma unroll
        for (int o = 0; o < kBW; ++o)
          if (pos[o] + st <= lim[o] && cand[o * kCapW + pos[o] + st - 1] > c) pos[o] += st;
      int rank = qi;
#pragma unroll
      for (int o = 0; o < kBW; ++o) rank += pos[o];
      if (rank < keff) ent[rank] = c;
      if (rank == keff - 1) reinterpret_cast<uint64_t*>(&ctl[6])[0] = c;  // the K-th
    }
    cbar();
    if (tid == 0) {
      float m = -INFINITY, Rp = -INFINITY;
      int bad = 0;
      uint64_t F = bounded ? make_comp(Tv, 0x7FFFFFFF) : 0;
      for (int w = 0; w < kBW; ++w) {
        m = fmaxf(m, parts[w].m);
        bad |= parts[w].bad;
        if (parts[w].s != 0.0) Rp = fmaxf(Rp, (float)parts[w].R);
        F = parts[w].floor > F ? parts[w].floor : F;
      }
      if (tot > keff) {
        const uint64_t kth = reinterpret_cast<uint64_t*>(&ctl[6])[0];
        F = kth > F ? kth : F;
      }
      double sv = 0.0;
      for (int w = 0; w < kBW; ++w)
        if (parts[w].s != 0.0) sv += parts[w].s * exp2(parts[w].R - (double)Rp);
      RecHdr h;
      h.m = m;
      h.flags = bad ? kRecBad : 0u;
      h.s = sv;
      h.R = (double)Rp;
      h.n = (uint32_t)n;
      h.rsv = 0;
      h.frontier = F;
      *reinterpret_cast<RecHdr*>(rec) = h;
      *tkey = 0;  // reset for the next piece
    }
    cbar();
    TRACE(ntr++);
    pos = pend;
  }
  TRACE(31);
}

// Phase B: one CTA per row merges the row's piece records (mode 0: final sample; mode 1: one
// merged record per row for the vocab-sharded exchange; world > 0: sharded phase 2, one record
// per rank).
struct MergeArgs {
  const uint8_t* records;
  int64_t rec_stride;
  int64_t span;
  int Vp;
  int V, kcand, mode;
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  int append;
  int pending_ok;
  HistState hs;
  RowOut ro;
  uint8_t* out_records;
  int64_t rank_pitch;
  int world;
};
constexpr int kMergeKernelSmem = kPool * 8 + 3 * SAMPLER_KCAND_MAX * 8 + kMaxRec * 48 + (kMaxRec + 1) * 4 + 12 + 512;

__global__ void __launch_bounds__(kBT) merge_rows_kernel(const MergeArgs m) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int r = blockIdx.x;
  MergeSmem ms;
  ms.pool = reinterpret_cast<uint64_t*>(smem);
  ms.top = reinterpret_cast<uint64_t*>(smem + kPool * 8);
  ms.wv = reinterpret_cast<double*>(smem + kPool * 8 + SAMPLER_KCAND_MAX * 8);
  ms.byid = reinterpret_cast<uint64_t*>(smem + kPool * 8 + 2 * SAMPLER_KCAND_MAX * 8);
  uint8_t* rest = smem + kPool * 8 + 3 * SAMPLER_KCAND_MAX * 8;
  ms.hdr = reinterpret_cast<RecHdr*>(rest);
  ms.off = reinterpret_cast<int*>(rest + kMaxRec * 48);
  uint8_t* scr = rest + kMaxRec * 48 + (kMaxRec + 1) * 4 + 12;
  scr = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(scr) + 15) & ~(uintptr_t)15);
  ms.bs.f = reinterpret_cast<float*>(scr);
  ms.bs.d = reinterpret_cast<double*>(scr + 32);
  ms.bs.u = reinterpret_cast<uint64_t*>(scr + 96);
  ms.bs.i = reinterpret_cast<int*>(scr + 224);
  const int slot = m.slots ? m.slots[r] : r;
  const sampling_params prm = m.params_dev ? m.params_dev[r] : m.params_tab[slot];
  const uint64_t seed = m.seeds ? m.seeds[r] : prm.seed;
  if (m.world > 0) {
    block_merge_row(m.records + (int64_t)r * m.rec_stride, m.rank_pitch, m.world, r, slot, prm, seed, m.step, m.V,
                    m.kcand, 0, nullptr, m.ro, m.append, m.hs, false, ms);
    return;
  }
  const int64_t c_first = ((int64_t)r * m.Vp) / m.span;
  const int64_t c_last = ((int64_t)(r + 1) * m.Vp - 1) / m.span;
  block_merge_row(m.records + (c_first + r) * m.rec_stride, m.rec_stride, (int)(c_last - c_first + 1), r, slot, prm,
                  seed, m.step, m.V, m.kcand, m.mode,
                  m.out_records ? m.out_records + (int64_t)r * m.rec_stride : nullptr, m.ro, m.append, m.hs,
                  m.pending_ok != 0, ms);
}

}  // namespace smp

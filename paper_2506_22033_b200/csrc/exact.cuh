// exact.cuh — exact multi-pass path for rows whose kept set is not bounded by the one-pass
// candidates (top-p / min-p-only rows with large nuclei, unfiltered rows, top_k > K_cand).
//
// One CTA (1024 threads) per pending row; M and S come from the streaming pass.
//   pass 0  materialise z' (penalties applied, binary32) into a per-row fp32 scratch row
//   pass 1  2048-bucket histogram of counts and fixed-point masses, bucket = floor(-x*64) with
//           x = (z'-M)*log2(e)/tau (1/64-octave buckets of the weight; contiguous in pi order)
//   select  top-k rank / top-p mass cutoffs: bucket by prefix scan, then inside the bucket by
//           gathering + sorting its composites (or, if it is huge, an 8-digit radix select)
//           min-p: exact value threshold by bisection on binary32 keys (w >= min_p, float64)
//   pass 2  draw: per-thread id-contiguous kept mass, block scan, inverse CDF in id order
// All reductions are integer (fixed point) or fixed-order float64: bit-reproducible.
#pragma once
#include "common.cuh"
#include "merge.cuh"
#include "philox.cuh"
#include "elem.cuh"

namespace smp {

constexpr int kExThreads = 1024;
constexpr int kNB = 2048;
constexpr int kCapG = 4096;
constexpr double kFix = 17592186044416.0;  // 2^44 fixed-point scale for masses (w <= 1)
constexpr int kExactSmem = kNB * 4 + kNB * 8 + kCapG * 8 + 1024 + 256 * 4 + 256 * 8;

struct ExactArgs {
  const void* logits;
  int64_t ld;
  int B, V, voff, vloc, Vp;
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  int append;
  int pen_mode;
  HistState hs;
  float* scratch;  // [B x Vp]
  RowOut ro;
};

struct ExSmem {
  uint32_t* cnt;   // [kNB]
  uint64_t* mass;  // [kNB]
  uint64_t* list;  // [kCapG]
  uint64_t* u64s;  // [32]
  double* dbl;     // [32]
  int* ints;       // [32]
  uint32_t* rcnt;  // [256] radix digit counts
  uint64_t* rmass; // [256] radix digit masses
};

__device__ __forceinline__ int bucket_of(float z, float M, float c_hi, float c_lo) {
  const float t = z - M;
  const float x = fmaf(t, c_hi, t * c_lo);
  const float y = -x * 64.0f;
  return y >= (float)(kNB - 1) ? kNB - 1 : (y > 0.0f ? (int)y : 0);
}

__device__ __forceinline__ uint64_t fixmass(float w) { return (uint64_t)__float2ull_rn(w * (float)kFix); }
// 64-bit shared-memory add as two native 32-bit atomics with the carry (sm_100 has no native
// 64-bit shared add: it would be a CAS spin loop); integer, so still order-independent
__device__ __forceinline__ void smem_add_u64(uint64_t* p, uint64_t v) {
  uint32_t* p32 = reinterpret_cast<uint32_t*>(p);
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(p32, lo);
  const uint32_t up = hi + ((uint32_t)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(p32 + 1, up);
}

// block-wide reductions (512 threads)
__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, ExSmem& s) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  __syncthreads();
  if (lane == 0) s.u64s[wid] = v;
  __syncthreads();
  uint64_t t = 0;
  for (int i = 0; i < kExThreads / 32; ++i) t += s.u64s[i];
  __syncthreads();
  return t;
}
__device__ __forceinline__ int block_sum_int(int v, ExSmem& s) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum_i(v);
  __syncthreads();
  if (lane == 0) s.ints[wid] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < kExThreads / 32; ++i) t += s.ints[i];
  __syncthreads();
  return t;
}
// exclusive scan of doubles in thread order (fixed order => deterministic); returns total
__device__ __forceinline__ double block_excl_scan_d(double v, double* total, ExSmem& s) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double incl = warp_incl_scan_d(v, lane);
  __syncthreads();
  if (lane == 31) s.dbl[wid] = incl;
  __syncthreads();
  double before = 0.0, tot = 0.0;
  for (int i = 0; i < kExThreads / 32; ++i) {
    if (i < wid) before += s.dbl[i];
    tot += s.dbl[i];
  }
  __syncthreads();
  *total = tot;
  return before + incl - v;
}

// First bucket b (ascending) where the running sum of `val` (count or mass, restricted to
// buckets < limit) reaches target; returns b (or -1) and the sum of buckets before b.
template <bool MASS>
__device__ int find_bucket(ExSmem& s, uint64_t target, int limit, uint64_t* before) {
  // each thread owns 4 consecutive buckets
  const int tid = threadIdx.x;
  uint64_t v[4];
  uint64_t loc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int b = tid * 4 + j;
    v[j] = (b < limit) ? (MASS ? s.mass[b] : (uint64_t)s.cnt[b]) : 0;
    loc += v[j];
  }
  // exclusive scan over threads (u64)
  const int lane = tid & 31, wid = tid >> 5;
  uint64_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) s.u64s[wid] = incl;
  __syncthreads();
  uint64_t wbefore = 0;
  for (int i = 0; i < wid; ++i) wbefore += s.u64s[i];
  uint64_t run = wbefore + incl - loc;
  __syncthreads();
  if (tid == 0) s.ints[0] = -1;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (run < target && run + v[j] >= target) {
      s.ints[0] = tid * 4 + j;
      s.u64s[0] = run;
    }
    run += v[j];
  }
  __syncthreads();
  const int b = s.ints[0];
  *before = (b >= 0) ? s.u64s[0] : 0;
  __syncthreads();
  return b;
}

// Descending bitonic sort of s.list[0..n) (n <= kCapG).
__device__ void block_sort_desc(ExSmem& s, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + threadIdx.x; i < N; i += kExThreads) s.list[i] = 0;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += kExThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s.list[i], b = s.list[ixj];
          const bool desc = (i & k) == 0;
          if (desc ? (a < b) : (a > b)) {
            s.list[i] = b;
            s.list[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

struct BucketCtx {
  const float* zs;  // scratch row
  int Vp, voff;
  float M, c_hi, c_lo;
};

// Gather the composites of bucket b (count nb <= kCapG) into s.list, sorted descending.
__device__ void gather_bucket(ExSmem& s, const BucketCtx& bc, int b, int nb) {
  if (threadIdx.x == 0) s.ints[1] = 0;
  __syncthreads();
  const float4* z4 = reinterpret_cast<const float4*>(bc.zs);
#pragma unroll 4
  for (int i = threadIdx.x; i < bc.Vp / 4; i += kExThreads) {
    const float4 q = z4[i];
    const float zz[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (zz[j] > -INFINITY && bucket_of(zz[j], bc.M, bc.c_hi, bc.c_lo) == b) {
        const int pos = atomicAdd(&s.ints[1], 1);
        if (pos < kCapG) s.list[pos] = make_comp(zz[j], bc.voff + i * 4 + j);
      }
    }
  }
  __syncthreads();
  block_sort_desc(s, nb);
}

// Radix select inside bucket b (any size): the cutoff composite C where the running count
// (or fixed-point mass) over the bucket's elements in descending composite order first
// reaches `target`.  8 digit passes over the row.
template <bool MASS>
__device__ uint64_t radix_in_bucket(ExSmem& s, const BucketCtx& bc, int b, uint64_t target,
                                   uint64_t floor_c = 0) {
  uint64_t prefix = 0;
  uint64_t need = target;
  for (int d = 56; d >= 0; d -= 8) {
    for (int i = threadIdx.x; i < 256; i += kExThreads) {
      s.rcnt[i] = 0;
      s.rmass[i] = 0;
    }
    __syncthreads();
#pragma unroll 4
    for (int i = threadIdx.x; i < bc.Vp; i += kExThreads) {
      const float z = bc.zs[i];
      if (!(z > -INFINITY) || bucket_of(z, bc.M, bc.c_hi, bc.c_lo) != b) continue;
      const uint64_t c = make_comp(z, bc.voff + i);
      if (c < floor_c) continue;
      if (d != 56 && (c >> (d + 8)) != prefix) continue;
      const int dig = (int)((c >> d) & 255);
      if (MASS) {
        const float t = z - bc.M;
        smem_add_u64(&s.rmass[dig], fixmass(ex2f(fmaf(t, bc.c_hi, t * bc.c_lo))));
      } else {
        atomicAdd(&s.rcnt[dig], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t run = 0;
      int pick = 0;
      for (int dg = 255; dg >= 0; --dg) {
        const uint64_t v = MASS ? s.rmass[dg] : (uint64_t)s.rcnt[dg];
        if (run + v >= need && v > 0) {
          pick = dg;
          break;
        }
        run += v;
        pick = dg;
      }
      s.ints[2] = pick;
      s.u64s[0] = run;
    }
    __syncthreads();
    const int pick = s.ints[2];
    need -= s.u64s[0];
    prefix = (prefix << 8) | (uint64_t)pick;
    __syncthreads();
  }
  return prefix;
}

template <typename T>
__global__ void __launch_bounds__(kExThreads, 1) exact_kernel(const __grid_constant__ ExactArgs a) {
  const int r = blockIdx.x;
  if (a.ro.info[r].status != kRowPending) return;
  extern __shared__ __align__(128) uint8_t smem[];
  ExSmem s;
  s.cnt = reinterpret_cast<uint32_t*>(smem);
  s.mass = reinterpret_cast<uint64_t*>(smem + kNB * 4);
  s.list = reinterpret_cast<uint64_t*>(smem + kNB * 12);
  s.u64s = reinterpret_cast<uint64_t*>(smem + kNB * 12 + kCapG * 8);
  s.dbl = reinterpret_cast<double*>(smem + kNB * 12 + kCapG * 8 + 256);
  s.ints = reinterpret_cast<int*>(smem + kNB * 12 + kCapG * 8 + 512);
  s.rcnt = reinterpret_cast<uint32_t*>(smem + kNB * 12 + kCapG * 8 + 1024);
  s.rmass = reinterpret_cast<uint64_t*>(smem + kNB * 12 + kCapG * 8 + 1024 + 1024);
  const int tid = threadIdx.x;
  const int slot = a.slots ? a.slots[r] : r;
  const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
  const RowCfg rc = decode_row(prm, a.V, 1);
  const RowInfo ri = a.ro.info[r];
  const float M = ri.M;
  const double S = ri.S;

  // ---- pass 0: z' row
  float* zs = a.scratch + (int64_t)r * a.Vp;
  const uint8_t* lrow = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * sizeof(T);
  {
    // 16-byte loads (8 bf16 / 4 f32 per vector; rows are 16-byte aligned, ld * elem % 16 == 0)
    constexpr int VEC = 16 / (int)sizeof(T);
    const int nvec = a.Vp / VEC;
#pragma unroll 4
    for (int v = tid; v < nvec; v += kExThreads) {
      const uint4 u = (v * VEC < a.vloc) ? *reinterpret_cast<const uint4*>(lrow + (int64_t)v * 16)
                                         : make_uint4(0u, 0u, 0u, 0u);
      float z[VEC];
      if (sizeof(T) == 2) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          z[2 * q] = __uint_as_float(w[q] << 16);
          z[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
        }
      } else {
        z[0] = __uint_as_float(u.x);
        z[1] = __uint_as_float(u.y);
        z[2] = __uint_as_float(u.z);
        z[3 % VEC] = __uint_as_float(u.w);
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (v * VEC + e >= a.vloc) z[e] = -INFINITY;
#pragma unroll
      for (int e = 0; e < VEC; e += 4)
        *reinterpret_cast<float4*>(zs + v * VEC + e) = make_float4(z[e], z[e + 1], z[e + 2], z[e + 3]);
    }
  }
  __syncthreads();
  {
    const UniqEntry* ut = a.hs.uniq + (int64_t)slot * a.hs.L;
    const int nu = a.hs.meta[slot].n_uniq;
    for (int i = tid; i < nu; i += kExThreads) {
      const UniqEntry e = ut[i];
      const int j = e.id - a.voff;
      if (j < 0 || j >= a.vloc) continue;
      float x;
      if (sizeof(T) == 2)
        x = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(lrow)[j] << 16);
      else
        x = reinterpret_cast<const float*>(lrow)[j];
      zs[j] = apply_penalty(x, e.meta, prm, a.pen_mode);
    }
  }
  __threadfence_block();
  __syncthreads();

  BucketCtx bc;
  bc.zs = zs;
  bc.Vp = a.Vp;
  bc.voff = a.voff;
  bc.M = M;
  bc.c_hi = rc.c_hi;
  bc.c_lo = rc.c_lo;

  // ---- pass 1: histogram
  for (int i = tid; i < kNB; i += kExThreads) {
    s.cnt[i] = 0;
    s.mass[i] = 0;
  }
  __syncthreads();
  int nfin_loc = 0;
  const float4* z4 = reinterpret_cast<const float4*>(zs);
#pragma unroll 4
  for (int i = tid; i < a.Vp / 4; i += kExThreads) {
    const float4 q = z4[i];
    const float zz[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (zz[j] > -INFINITY) {
        const float t = zz[j] - M;
        const float x = fmaf(t, rc.c_hi, t * rc.c_lo);
        const float y = -x * 64.0f;
        const int b = y >= (float)(kNB - 1) ? kNB - 1 : (y > 0.0f ? (int)y : 0);
        atomicAdd(&s.cnt[b], 1u);
        smem_add_u64(&s.mass[b], fixmass(ex2f(x)));
        ++nfin_loc;
      }
    }
  }
  __syncthreads();
  const int nfin = block_sum_int(nfin_loc, s);

  // ---- cutoffs (composites; K = {composite >= C})
  uint64_t Ck = 0, Cp = 0, Cm = 0;
  int bk = kNB;          // bucket holding the k-th element (kNB: top-k off / keeps all)
  double W1 = 0.0;
  bool k_sorted = false;  // s.list holds bucket bk sorted
  int nbk = 0;
  if (rc.topk_on && rc.k < nfin) {
    uint64_t before;
    bk = find_bucket<false>(s, (uint64_t)rc.k, kNB, &before);
    nbk = (int)s.cnt[bk];
    const int need = rc.k - (int)before;
    if (nbk <= kCapG) {
      gather_bucket(s, bc, bk, nbk);
      Ck = s.list[need - 1];
      k_sorted = true;
    } else {
      Ck = radix_in_bucket<false>(s, bc, bk, (uint64_t)need);
    }
  }
  if (rc.top_p < 1.0f) {
    // W1 = mass of K1
    if (bk < kNB) {
      uint64_t mabove = 0;
      for (int b = tid; b < bk; b += kExThreads) mabove += s.mass[b];
      mabove = block_sum_u64(mabove, s);
      double part = 0.0;
      if (k_sorted) {
        double loc = 0.0;
        for (int i = tid; i < nbk; i += kExThreads)
          if (s.list[i] >= Ck) loc += exp(((double)comp_val(s.list[i]) - (double)M) / (double)rc.tau);
        double tot;
        block_excl_scan_d(loc, &tot, s);
        part = tot;
      } else {
        // partial mass inside bk via a pass
        double loc = 0.0;
#pragma unroll 4
        for (int i = tid; i < a.Vp; i += kExThreads) {
          const float z = zs[i];
          if (z > -INFINITY && bucket_of(z, M, rc.c_hi, rc.c_lo) == bk && make_comp(z, a.voff + i) >= Ck) {
            const float t = z - M;
            loc += (double)ex2f(fmaf(t, rc.c_hi, t * rc.c_lo));
          }
        }
        double tot;
        block_excl_scan_d(loc, &tot, s);
        part = tot;
      }
      W1 = (double)mabove / kFix + part;
    } else {
      W1 = S;
    }
    const double target = (double)rc.top_p * W1;
    const uint64_t tfix = (uint64_t)(target * kFix);
    uint64_t before;
    const int bp = find_bucket<true>(s, tfix > 0 ? tfix : 1, bk, &before);
    if (bp >= 0) {
      const int nb = (int)s.cnt[bp];
      if (nb <= kCapG) {
        gather_bucket(s, bc, bp, nb);
        // walk in pi order with float64 weights: first i with before + c_i >= target
        double lw = 0.0;
        // each thread: contiguous run of the sorted list
        const int per = (nb + kExThreads - 1) / kExThreads;
        const int i0 = tid * per, i1 = min(nb, i0 + per);
        for (int i = i0; i < i1; ++i) lw += exp(((double)comp_val(s.list[i]) - (double)M) / (double)rc.tau);
        double tot;
        const double ex = block_excl_scan_d(lw, &tot, s) + (double)before / kFix;
        if (tid == 0) s.ints[3] = nb - 1;
        __syncthreads();
        double run = ex;
        for (int i = i0; i < i1; ++i) {
          run += exp(((double)comp_val(s.list[i]) - (double)M) / (double)rc.tau);
          if (run >= target) {
            atomicMin(&s.ints[3], i);
            break;
          }
        }
        __syncthreads();
        Cp = s.list[s.ints[3]];
        __syncthreads();
      } else {
        const uint64_t need = tfix - before;
        Cp = radix_in_bucket<true>(s, bc, bp, need > 0 ? need : 1);
      }
    } else if (bk < kNB) {
      // cutoff falls inside the top-k boundary bucket (or rounding shortfall): walk K1's part
      if (k_sorted) {
        uint64_t mabove = 0;
        for (int b = tid; b < bk; b += kExThreads) mabove += s.mass[b];
        mabove = block_sum_u64(mabove, s);
        if (tid == 0) {
          double run = (double)mabove / kFix;
          uint64_t pick = Ck;
          for (int i = 0; i < nbk && s.list[i] >= Ck; ++i) {
            run += exp(((double)comp_val(s.list[i]) - (double)M) / (double)rc.tau);
            if (run >= target) {
              pick = s.list[i];
              break;
            }
          }
          s.u64s[1] = pick;
        }
        __syncthreads();
        Cp = s.u64s[1];
        __syncthreads();
      } else {
        uint64_t mabove = 0;
        for (int b = tid; b < bk; b += kExThreads) mabove += s.mass[b];
        mabove = block_sum_u64(mabove, s);
        const uint64_t need = tfix > mabove ? tfix - mabove : 1;
        Cp = radix_in_bucket<true>(s, bc, bk, need, Ck);
        if (Cp < Ck) Cp = Ck;
      }
    }
  }
  if (rc.min_p > 0.0f) {
    // smallest binary32 z with exp((z-M)/tau) >= min_p  (bisection on monotone keys)
    if (tid == 0) {
      uint32_t lo = f2key(-INFINITY), hi = f2key(M);  // w(hi) = 1 >= min_p
      while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        const double z = (double)key2f(mid);
        if (exp((z - (double)M) / (double)rc.tau) >= (double)rc.min_p)
          hi = mid;
        else
          lo = mid;
      }
      s.u64s[2] = ((uint64_t)hi << 32);  // every id with value >= key2f(hi)
    }
    __syncthreads();
    Cm = s.u64s[2];
    __syncthreads();
  }
  uint64_t C3 = Ck;
  C3 = Cp > C3 ? Cp : C3;
  C3 = Cm > C3 ? Cm : C3;

  // ---- pass 2: draw in ascending id order over K3 = {composite >= C3}
  // (each thread owns a contiguous, 16-byte aligned id range: Vp is a multiple of 4)
  const int per = ((a.Vp + kExThreads - 1) / kExThreads + 3) / 4 * 4;
  const int j0 = min(a.Vp, tid * per), j1 = min(a.Vp, j0 + per);
  double loc = 0.0;
#pragma unroll 2
  for (int j = j0; j < j1; j += 4) {
    const float4 q = *reinterpret_cast<const float4*>(zs + j);
    const float zz[4] = {q.x, q.y, q.z, q.w};
    float l4 = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (zz[e] > -INFINITY && make_comp(zz[e], a.voff + j + e) >= C3) {
        const float t = zz[e] - M;
        l4 += ex2f(fmaf(t, rc.c_hi, t * rc.c_lo));
      }
    loc += (double)l4;
  }
  double W;
  const double ex = block_excl_scan_d(loc, &W, s);
  const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
  const double u = philox_uniform(seed, prm.request_id, a.step);
  const double target = u * W;
  if (tid == 0) s.ints[4] = 0x7FFFFFFF;
  __syncthreads();
  if (ex <= target && target < ex + loc) {
    // the same arithmetic as the chunk sum above: float sums of 4, then float64
    double run = ex;
    for (int j = j0; j < j1; j += 4) {
      float w4[4], l4 = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float z = zs[j + e];
        w4[e] = 0.f;
        if (z > -INFINITY && make_comp(z, a.voff + j + e) >= C3) {
          const float t = z - M;
          w4[e] = ex2f(fmaf(t, rc.c_hi, t * rc.c_lo));
        }
        l4 += w4[e];
      }
      if (run + (double)l4 > target) {
        float cf = 0.f;
        int pick = j + 3;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          cf += w4[e];
          if (w4[e] > 0.f && run + (double)cf > target) {
            pick = j + e;
            break;
          }
        }
        atomicMin(&s.ints[4], pick);
        break;
      }
      run += (double)l4;
    }
  }
  __syncthreads();
  int jt = s.ints[4];
  if (jt == 0x7FFFFFFF) {
    // rounding: take the last kept id
    int last = -1;
    for (int j = j0; j < j1; ++j)
      if (zs[j] > -INFINITY && make_comp(zs[j], a.voff + j) >= C3) last = j;
    __syncthreads();
    if (tid == 0) s.ints[4] = -1;
    __syncthreads();
    atomicMax(&s.ints[4], last);
    __syncthreads();
    jt = s.ints[4];
  }
  if (tid == 0) {
    const float zt = zs[jt];
    const double wt = exp(((double)zt - (double)M) / (double)rc.tau);
    const double lp = ((double)zt - (double)M) / (double)rc.tau - log(S);
    const int32_t tok = a.voff + jt;
    a.ro.tokens[r] = tok;
    a.ro.logprobs[r] = (float)lp;
    if (a.ro.flogprobs) a.ro.flogprobs[r] = (float)log(wt / W);
    if (a.ro.status) a.ro.status[r] = SAMPLER_ROW_OK;
    RowInfo o = ri;
    o.status = SAMPLER_ROW_OK;
    o.W = W;
    o.cutoff = C3;
    o.token = tok;
    a.ro.info[r] = o;
    s.ints[5] = tok;
  }
  __syncthreads();
  if (a.append && tid < 32) warp_append_token(a.hs, slot, s.ints[5], tid);
}

// Debug: q[b, v] = final filtered distribution (w_v / W over K3; one-hot for greedy rows).
template <typename T>
__global__ void debug_q_kernel(const void* logits, int64_t ld, int V, int voff, int vloc,
                               const int32_t* slots, const sampling_params* params_dev,
                               const sampling_params* params_tab, int pen_mode, HistState hs,
                               const RowInfo* info, float* q) {
  const int r = blockIdx.y;
  const RowInfo ri = info[r];
  const int slot = slots ? slots[r] : r;
  const sampling_params prm = params_dev ? params_dev[r] : params_tab[slot];
  const RowCfg rc = decode_row(prm, V, 1);
  const UniqEntry* ut = hs.uniq + (int64_t)slot * hs.L;
  const int nu = hs.meta[slot].n_uniq;
  const uint8_t* lrow = reinterpret_cast<const uint8_t*>(logits) + (int64_t)r * ld * sizeof(T);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < vloc; j += gridDim.x * blockDim.x) {
    float out = 0.0f;
    if (ri.status == SAMPLER_ROW_OK) {
      if (ri.greedy) {
        out = (voff + j == ri.token) ? 1.0f : 0.0f;
      } else {
        float x = sizeof(T) == 2
                      ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(lrow)[j] << 16)
                      : reinterpret_cast<const float*>(lrow)[j];
        // penalty lookup (binary search; debug only)
        int lo = 0, hi = nu;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (ut[mid].id < voff + j) lo = mid + 1; else hi = mid;
        }
        if (lo < nu && ut[lo].id == voff + j) x = apply_penalty(x, ut[lo].meta, prm, pen_mode);
        if (x > -INFINITY && make_comp(x, voff + j) >= ri.cutoff)
          out = (float)(exp(((double)x - (double)ri.M) / (double)rc.tau) / ri.W);
      }
    } else {
      out = NAN;
    }
    q[(int64_t)r * V + voff + j] = out;
  }
}

}  // namespace smp

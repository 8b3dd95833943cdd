// exact.cuh — the exact path for rows whose kept set is not bounded by the one-pass candidates
// (top-p / min-p-only rows with large nuclei, unfiltered rows, top_k > K_cand).
//
// One thread-block cluster of G CTAs per row (G = 1 for large batches); CTA c takes the chunk
// [c*Lc, (c+1)*Lc) of the row's vocabulary slice and reads it from global memory (L2) in every pass;
// M (row max of z') and S come from phase B (select.cuh).  Every mass is float64-accurate (DESIGN.md
// R16: a token may differ from the oracle's only when a boundary lies within 1e-9 of it):
//   pass 1  per element y = (M - z') log2(e)/tau >= 0 (float64), weight w = 2^-y
//           (= exp((z' - M)/tau)), bucket b = floor(64 y) (1/64 octave of weight, so buckets
//           are contiguous in pi order); per bucket its count and its mass RELATIVE TO THE BUCKET'S
//           TOP WEIGHT 2^(-b/64), in 2^-40 fixed point: sum_i round(2^(b/64 - y_i) 2^40), each term in
//           (2^39.98, 2^40], so every element keeps <= 2^-41 relative error and the sums are
//           order-independent integers (deterministic).  The leader CTA sums the C histograms.
//   cutoffs top-k (count) and top-p (mass over K1, P:149's Filter; R7/R8) locate their
//           bucket from the fixed-order prefix of the bucket masses, then gather that bucket's
//           elements (all CTAs -> the leader, DSMEM), sort them by (z' desc, id asc) and walk them
//           with exact float64 weights; a bucket too large to gather is split once more into 1024
//           sub-buckets (1/65536 octave); min-p is an exact value threshold (bisection, float64).
//   draw    K3 = { composite >= C3 }; W = sum over K3 of w in id order: per-CTA totals, the
//           cluster prefix in CTA (= id) order, u*W located, the CTA holding it walks its chunk in
//           id order (rounds of 512 vectors, block scans): first cumulative > u*W.
#pragma once
#include <cfloat>

#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "philox.cuh"
#include "piece.cuh"

namespace smp {

constexpr int kExThreads = 512;
constexpr int kExW = kExThreads / 32;
constexpr int kNB0 = 2048;   // level-0 buckets: 1/64 octave, 32 octaves
constexpr int kNB1 = 1024;   // level-1 sub-buckets of one level-0 bucket: 1/65536 octave
constexpr int kSide = 2048;  // penalised (local id, z') of the chunk kept in smem
constexpr int kGat = 4096;   // gathered composites of the boundary bucket (leader)
constexpr double kFix40 = 1099511627776.0;  // 2^40

struct ExactArgs {
  const void* logits;
  int64_t ld;
  int B, V, voff, vloc;
  int G, Lc;  // cluster size, chunk length (multiple of 128)
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  int append;
  int pen_mode;
  HistState hs;
  RowOut ro;
};

// shared memory (bytes)
constexpr int kExOffSideId = 0;
constexpr int kExOffSideZ = kExOffSideId + kSide * 4;
constexpr int kExOffCnt = kExOffSideZ + kSide * 4;     // u32 [kNB0] local counts
constexpr int kExOffMass = kExOffCnt + kNB0 * 4;       // u64 [kNB0] local fixed masses
constexpr int kExOffGat = kExOffMass + kNB0 * 8;       // u64 [kGat] (leader)
constexpr int kExOffWt = kExOffGat + kGat * 8;         // double [kNB0] 2^(-b/64)
constexpr int kExOffScr = kExOffWt + kNB0 * 8;         // scratch: doubles / ints / u64
constexpr int kExactSmem = kExOffScr + 2048;

// ---- cluster helpers (a launch without clusters is a cluster of one CTA) ----------------
__device__ __forceinline__ uint32_t ex_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void ex_csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ex_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ex_ld32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a));  // (ordered by cluster barriers)
  return v;
}
__device__ __forceinline__ uint64_t ex_ld64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void ex_st64(uint32_t a, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ex_atom_add(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void ex_bar() { __syncthreads(); }

// 64-bit shared-memory add as two native 32-bit atomics with the carry (integer: order-independent)
__device__ __forceinline__ void smem_add_u64(uint64_t* p, uint64_t v) {
  uint32_t* p32 = reinterpret_cast<uint32_t*>(p);
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(p32, lo);
  const uint32_t up = hi + ((uint32_t)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(p32 + 1, up);
}

// 2^-s for s in [0, ln2/64) via its series in s*ln2 (relative error < 3e-15)
__device__ __forceinline__ double exp2_neg_small(double d) {  // d = s * ln2 in [0, 0.0109)
  return 1.0 - d * (1.0 - d * (0.5 - d * (1.0 / 6.0 - d * (1.0 / 24.0 - d * (1.0 / 120.0)))));
}

// block-wide fixed-order sums / scans (512 threads)
__device__ __forceinline__ double ex_sum_d(double v, double* scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum_d(v);
  ex_bar();
  if (lane == 0) scr[w] = v;
  ex_bar();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kExW; ++i) t += scr[i];
  ex_bar();
  return t;
}
__device__ __forceinline__ double ex_excl_scan_d(double v, double* tot, double* scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double incl = warp_incl_scan_d(v, lane);
  ex_bar();
  if (lane == 31) scr[w] = incl;
  ex_bar();
  double before = 0.0, t = 0.0;
#pragma unroll
  for (int i = 0; i < kExW; ++i) {
    if (i < w) before += scr[i];
    t += scr[i];
  }
  ex_bar();
  *tot = t;
  return before + incl - v;
}
__device__ __forceinline__ uint64_t ex_sum_u64(uint64_t v, uint64_t* scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  ex_bar();
  if (lane == 0) scr[w] = v;
  ex_bar();
  uint64_t t = 0;
#pragma unroll
  for (int i = 0; i < kExW; ++i) t += scr[i];
  ex_bar();
  return t;
}

// Descending bitonic sort of buf[0..n) (n <= kGat) by the whole block.
__device__ void ex_sort_desc(uint64_t* buf, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + threadIdx.x; i < N; i += kExThreads) buf[i] = 0;
  ex_bar();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += kExThreads) {
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
      ex_bar();
    }
}

// the row as seen by one CTA: z' of local id l (penalties applied), element iteration by vectors
template <typename T>
struct ExRow {
  static constexpr int VEC = Dec<T>::N;
  const uint8_t* rowp;      // local slice of the row
  const uint32_t* pm;       // the slot's presence bitmap (phase A step-lane layout)
  const int* side_id;       // sorted local ids of the chunk's penalised elements
  const float* side_z;
  int nside;                // entries in smem (if ovf: the chunk's penalised ids come from the table)
  bool ovf;
  const UniqEntry* ut;      // the slot's unique-token table (sorted by id)
  int nu;
  int voff, vloc, c0, c1;   // chunk [c0, c1) of local ids
  sampling_params prm;
  int pen_mode;
  // penalised bits of vector v (VEC elements at local id v*VEC)
  __device__ __forceinline__ uint32_t pbits(int v) const {
    const int k = v >> 7, d = v & 127;
    return (pm[k * 32 + (d & 31)] >> ((d >> 5) * VEC)) & ((1u << VEC) - 1u);
  }
  __device__ __forceinline__ float pen_value(int l) const {
    if (!ovf) {
      int lo = 0, hi = nside;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (side_id[mid] < l) lo = mid + 1;
        else hi = mid;
      }
      return side_z[lo];
    }
    const int id = voff + l;
    int lo = 0, hi = nu;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ut[mid].id < id) lo = mid + 1;
      else hi = mid;
    }
    return apply_penalty(Dec<T>::load1(rowp, l), ut[lo].meta, prm, pen_mode);
  }
  // the VEC values z' of vector v (-inf past the slice end)
  __device__ __forceinline__ void vec(int v, float (&z)[Dec<T>::N]) const {
    const uint4 u = *reinterpret_cast<const uint4*>(rowp + (int64_t)v * 16);
    const uint32_t pb = pbits(v);
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      const int l = v * VEC + t;
      z[t] = (l < c1) ? Dec<T>::elem(u, t) : -INFINITY;
      if ((pb >> t) & 1u) z[t] = (l < c1) ? pen_value(l) : -INFINITY;
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(kExThreads, 1) exact_kernel(const __grid_constant__ ExactArgs a) {
  constexpr int VEC = Dec<T>::N;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x;
  const uint32_t rank = ex_rank();
  const int r = blockIdx.x / a.G;
  const RowInfo ri = a.ro.info[r];
  if (ri.status != kRowPending) return;  // (uniform over the cluster: no CTA of it continues)
  int* side_id = reinterpret_cast<int*>(smem + kExOffSideId);
  float* side_z = reinterpret_cast<float*>(smem + kExOffSideZ);
  uint32_t* hcnt = reinterpret_cast<uint32_t*>(smem + kExOffCnt);
  uint64_t* hmass = reinterpret_cast<uint64_t*>(smem + kExOffMass);
  uint64_t* gat = reinterpret_cast<uint64_t*>(smem + kExOffGat);
  double* sd = reinterpret_cast<double*>(smem + kExOffScr);        // [32]
  uint64_t* su = reinterpret_cast<uint64_t*>(smem + kExOffScr + 256);  // [32]
  int* si = reinterpret_cast<int*>(smem + kExOffScr + 512);           // [64]
  // control block (written by the leader into every CTA): [0] phase-specific ints, doubles at sd2
  int* ctl = reinterpret_cast<int*>(smem + kExOffScr + 768);          // [32]
  double* cd = reinterpret_cast<double*>(smem + kExOffScr + 896);     // [16]
  uint64_t* cu = reinterpret_cast<uint64_t*>(smem + kExOffScr + 1024);  // [16]
  double* tots = reinterpret_cast<double*>(smem + kExOffScr + 1152);    // [16] per-CTA draw totals (leader)
  double* wtab = reinterpret_cast<double*>(smem + kExOffWt);             // [kNB0] bucket top weights
  for (int b = tid; b < kNB0; b += kExThreads) wtab[b] = exp2(-(double)b / 64.0);

  const int slot = row_slot(a.slots, r, a.hs.nslots, nullptr);  // (pending rows have a valid slot)
  const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
  const RowCfg rc = decode_row(prm, a.V, 1);
  const float M = ri.M;
  const double inv_tau = 1.0 / (double)rc.tau;
  const double l2e_tau = kLog2e / (double)rc.tau;

  ExRow<T> R;
  R.rowp = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * sizeof(T);
  R.pm = a.hs.pmask + (int64_t)slot * a.hs.spr * 32;
  R.side_id = side_id;
  R.side_z = side_z;
  R.ut = a.hs.uniq + (int64_t)slot * a.hs.L;
  R.nu = a.hs.meta[slot].n_uniq;
  R.voff = a.voff;
  R.vloc = a.vloc;
  R.c0 = min(a.vloc, (int)rank * a.Lc);
  R.c1 = min(a.vloc, R.c0 + a.Lc);
  R.prm = prm;
  R.pen_mode = a.pen_mode;
  const int v0 = R.c0 / VEC, v1 = (R.c1 + VEC - 1) / VEC;  // vectors of the chunk

  // ---- the chunk's penalised elements: their table entries are contiguous (sorted by id)
  {
    int below = 0, inside = 0;
    for (int e = tid; e < R.nu; e += kExThreads) {
      const int l = R.ut[e].id - a.voff;
      below += (l < R.c0) ? 1 : 0;
      inside += (l >= R.c0 && l < R.c1) ? 1 : 0;
    }
    const int lo = (int)ex_sum_u64((uint64_t)below, su), n = (int)ex_sum_u64((uint64_t)inside, su);
    R.ovf = n > kSide;
    R.nside = R.ovf ? 0 : n;
    for (int e = tid; e < R.nside; e += kExThreads) {
      const UniqEntry ue = R.ut[lo + e];
      const int l = ue.id - a.voff;
      side_id[e] = l;
      side_z[e] = apply_penalty(Dec<T>::load1(R.rowp, l), ue.meta, prm, a.pen_mode);
    }
  }
  // weight coordinates of z: y = (M - z) log2(e)/tau; w = 2^-y; level-0 bucket floor(64 y)
  auto ycoord = [&](float z) -> double { return ((double)M - (double)z) * l2e_tau; };
  // w = exp((z - M)/tau) = 2^-y = 2^(-b/64) * 2^-(y - b/64): the bucket top from the table, the
  // rest by its short series (relative error < 3e-15); the far tail (y >= 32) directly
  auto weight = [&](float z) -> double {
    const double y = ycoord(z);
    const int b = (int)(y * 64.0);
    if (b >= kNB0 - 1) return exp2(-y);
    return wtab[b] * exp2_neg_small((y - (double)b / 64.0) * kLn2);
  };
  // one pass over the chunk's elements (coalesced: vector v of thread tid, stride 512)
  auto for_each = [&](auto&& fn) {
    for (int v = v0 + tid; v < v1; v += kExThreads) {
      float z[VEC];
      R.vec(v, z);
#pragma unroll
      for (int t = 0; t < VEC; ++t)
        if (z[t] > -INFINITY) fn(z[t], v * VEC + t);
    }
  };
  // histogram of a level: bucket(y) in [0, nb) for y in [ybase, ybase + nb / scale), masses
  // relative to the bucket top 2^-(ybase + b/scale)
  auto histogram = [&](double ybase, double scale, int nb) {
    for (int i = tid; i < nb; i += kExThreads) {
      hcnt[i] = 0;
      hmass[i] = 0;
    }
    ex_bar();
    for_each([&](float z, int) {
      const double y = ycoord(z);
      const double q = (y - ybase) * scale;
      if (!(q >= 0.0)) return;
      int b = (int)q;
      if (b >= nb) {
        if (nb == kNB0) b = nb - 1;  // (level 0: the far tail shares the last bucket)
        else return;
      }
      const double d = (y - ybase - (double)b / scale) * kLn2;  // >= 0
      const double rel = (b == nb - 1 && nb == kNB0) ? exp2(-(y - ybase - (double)b / scale)) : exp2_neg_small(d);
      atomicAdd(&hcnt[b], 1u);
      smem_add_u64(&hmass[b], (uint64_t)(rel * kFix40 + 0.5));
    });
    ex_bar();
  };
  // the cluster's total of bucket b (leader; reads every CTA's histogram over DSMEM)
  auto tot_bucket = [&](int b, uint32_t* cnt, uint64_t* mass) {
    uint32_t cv[8];
    uint64_t mv[8];
#pragma unroll
    for (int g = 0; g < 8; ++g)  // (all loads in flight, then the sums in CTA order)
      if (g < a.G) {
        cv[g] = ex_ld32(ex_map(hcnt + b, (uint32_t)g));
        mv[g] = ex_ld64(ex_map(hmass + b, (uint32_t)g));
      }
    uint32_t c = 0;
    uint64_t m = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (g < a.G) {
        c += cv[g];
        m += mv[g];
      }
    *cnt = c;
    *mass = m;
  };
  // gather the composites of every element of bucket b (level given) into the leader's buffer
  auto gather = [&](double ybase, double scale, int nb, int b) {
    const uint32_t cnt_addr = ex_map(ctl + 20, 0);
    for_each([&](float z, int l) {
      const double q = (ycoord(z) - ybase) * scale;
      if (!(q >= 0.0)) return;
      int bb = (int)q;
      if (bb >= nb) {
        if (nb == kNB0) bb = nb - 1;
        else return;
      }
      if (bb != b) return;
      const uint32_t at = ex_atom_add(cnt_addr, 1u);
      if (at < (uint32_t)kGat) ex_st64(ex_map(gat + at, 0), make_comp(z, a.voff + l));
    });
  };

  ex_csync();  // every CTA's side list is built; the cluster is resident
  // ---- pass 1: level-0 histograms; the leader sums the cluster's and finds the cutoffs
  histogram(0.0, 64.0, kNB0);
  ex_csync();
  // level-0 totals per bucket, in the leader; every CTA reads them (fixed order, deterministic)
  uint32_t tc[kNB0 / kExThreads];
  double tm[kNB0 / kExThreads];
  for (int j = 0; j < kNB0 / kExThreads; ++j) {
    const int b = tid * (kNB0 / kExThreads) + j;  // thread owns 4 consecutive buckets
    uint64_t m;
    tot_bucket(b, &tc[j], &m);
    tm[j] = (double)m * (1.0 / kFix40) * exp2(-(double)b / 64.0);
  }
  ex_csync();  // (every CTA has read every histogram; they may be reused)

  // cutoffs as composites: K = { composite >= C }
  uint64_t Ck = 0, Cp = 0, Cm = 0;
  double W1 = 0.0;
  // bucket-level prefix (counts, masses) in bucket order = pi order
  uint32_t cloc = 0;
  double mloc = 0.0;
  for (int j = 0; j < kNB0 / kExThreads; ++j) {
    cloc += tc[j];
    mloc += tm[j];
  }
  const uint64_t nfin = ex_sum_u64((uint64_t)cloc, su);
  double mtot;
  const double mbefore = ex_excl_scan_d(mloc, &mtot, sd);
  // exclusive count prefix per thread (integer)
  uint32_t cb;
  {
    const int lane = tid & 31, w = tid >> 5;
    const int incl = warp_incl_scan_i((int)cloc, lane);
    ex_bar();
    if (lane == 31) si[w] = incl;
    ex_bar();
    int bf = 0;
    for (int i = 0; i < w; ++i) bf += si[i];
    cb = (uint32_t)(bf + incl - (int)cloc);
    ex_bar();
  }
  const bool topk = rc.topk_on && (uint64_t)rc.k < nfin;
  // locate the bucket where a running quantity (count or mass) first reaches target
  auto find_bucket = [&](bool mass, double target, uint64_t ctarget, int limit, int* bucket, double* before) {
    if (tid == 0) ctl[0] = 0x7FFFFFFF;
    ex_bar();
    double run = mbefore;
    uint32_t crun = cb;
    for (int j = 0; j < kNB0 / kExThreads; ++j) {
      const int b = tid * (kNB0 / kExThreads) + j;
      if (b >= limit) break;
      const bool hit = mass ? (run + tm[j] >= target) : ((uint64_t)crun + tc[j] >= ctarget);
      if (hit && tc[j] > 0) {
        atomicMin(&ctl[0], b);  // (the first bucket reaching the target)
      }
      run += tm[j];
      crun += tc[j];
    }
    ex_bar();
    const int bsel = ctl[0] == 0x7FFFFFFF ? -1 : ctl[0];
    // its prefix: recompute in fixed order from the per-thread values (the owner publishes it)
    ex_bar();
    if (bsel >= 0 && tid == bsel / (kNB0 / kExThreads)) {
      double rr = mbefore;
      uint32_t cr = cb;
      for (int j = 0; j < bsel - tid * (kNB0 / kExThreads); ++j) {
        rr += tm[j];
        cr += tc[j];
      }
      cd[0] = rr;
      ctl[1] = (int)cr;
      cd[1] = tm[bsel - tid * (kNB0 / kExThreads)];
      ctl[2] = (int)tc[bsel - tid * (kNB0 / kExThreads)];
    }
    ex_bar();
    *bucket = bsel;
    *before = mass ? cd[0] : (double)ctl[1];
    ex_bar();
  };
  // exact resolution inside bucket b0 of level 0: gather its elements (or, if too many, those of
  // the level-1 sub-bucket reaching the target), sort by (z' desc, id asc) and walk with exact w.
  // mode 0: the count-th element (count = need); mode 1: the first element whose cumulative mass
  // (from `before`) reaches target; returns its composite and the exact mass of the walked prefix.
  auto resolve = [&](int b0, int mode, uint64_t need, double before, double target, double* prefix_mass) -> uint64_t {
    double ybase = (double)b0 / 64.0, scale = 65536.0;
    int level = 0;
    if (tid == 0) ctl[20] = 0;
    ex_csync();
    gather(0.0, 64.0, kNB0, b0);
    ex_csync();
    if (ctl[20] == 0 || rank != 0) {
      // (non-leaders only help gather)
    }
    int n = (int)ex_ld32(ex_map(ctl + 20, 0));
    ex_csync();
    if (n > kGat) {  // too large: one more level inside bucket b0
      level = 1;
      histogram(ybase, scale, kNB1);
      ex_csync();
      // leader: the sub-bucket; every CTA computes the same from the cluster totals
      uint32_t sc[kNB1 / kExThreads];
      double sm[kNB1 / kExThreads];
      for (int j = 0; j < kNB1 / kExThreads; ++j) {
        const int b = tid * (kNB1 / kExThreads) + j;
        uint64_t m;
        tot_bucket(b, &sc[j], &m);
        sm[j] = (double)m * (1.0 / kFix40) * exp2(-(ybase + (double)b / scale));
      }
      ex_csync();
      double l_m = 0.0;
      uint32_t l_c = 0;
      for (int j = 0; j < kNB1 / kExThreads; ++j) {
        l_m += sm[j];
        l_c += sc[j];
      }
      double dummy;
      const double mb = ex_excl_scan_d(l_m, &dummy, sd) + before;
      uint32_t cbb;
      {
        const int lane = tid & 31, w = tid >> 5;
        const int incl = warp_incl_scan_i((int)l_c, lane);
        ex_bar();
        if (lane == 31) si[w] = incl;
        ex_bar();
        int bf = 0;
        for (int i = 0; i < w; ++i) bf += si[i];
        cbb = (uint32_t)(bf + incl - (int)l_c);
        ex_bar();
      }
      if (tid == 0) ctl[0] = 0x7FFFFFFF;
      ex_bar();
      {
        double rr = mb;
        uint32_t cr = cbb;
        for (int j = 0; j < kNB1 / kExThreads; ++j) {
          const int b = tid * (kNB1 / kExThreads) + j;
          const bool hit = (mode == 1) ? (rr + sm[j] >= target) : ((uint64_t)cr + sc[j] >= need);
          if (hit && sc[j] > 0) atomicMin(&ctl[0], b);
          rr += sm[j];
          cr += sc[j];
        }
      }
      ex_bar();
      int sb = ctl[0];
      if (sb == 0x7FFFFFFF) sb = kNB1 - 1;
      ex_bar();
      if (tid == sb / (kNB1 / kExThreads)) {
        double rr = mb;
        uint32_t cr = cbb;
        for (int j = 0; j < sb - tid * (kNB1 / kExThreads); ++j) {
          rr += sm[j];
          cr += sc[j];
        }
        cd[2] = rr;
        ctl[3] = (int)cr;
      }
      ex_bar();
      before = cd[2];
      const uint64_t cbefore = (uint64_t)ctl[3];
      if (mode == 0) need -= (cbefore - 0);  // (need counted from the bucket start)
      ex_bar();
      if (tid == 0) ctl[20] = 0;
      ex_csync();
      gather(ybase, scale, kNB1, sb);
      ex_csync();
      n = (int)ex_ld32(ex_map(ctl + 20, 0));
      ex_csync();
    }
    n = min(n, kGat);  // (beyond: a pathological tie mass; the first kGat are kept)
    uint64_t pick = 0;
    double pm = before;
    if (rank == 0) {
      ex_sort_desc(gat, n);
      // walk the sorted bucket with exact float64 weights: rounds of 512 entries, block scans in
      // sorted (= pi) order; the first entry whose cumulative count / mass reaches the target
      if (tid == 0) {
        ctl[13] = 0x7FFFFFFF;
        cu[0] = n > 0 ? gat[n - 1] : 0;
        cd[3] = before;
      }
      ex_bar();
      double run = before;
      for (int i0 = 0; i0 < n; i0 += kExThreads) {
        const int i = i0 + tid;
        const double w = (i < n) ? weight(comp_val(gat[i])) : 0.0;
        double rt;
        const double c = ex_excl_scan_d(w, &rt, sd) + run + w;  // inclusive cumulative of entry i
        const bool hit = i < n && (mode == 0 ? ((uint64_t)(i + 1) >= need) : (c >= target));
        if (hit) atomicMin(&ctl[13], i);
        ex_bar();
        const int first = ctl[13];
        if (first != 0x7FFFFFFF) {
          if (i == first) {
            cu[0] = gat[i];
            cd[3] = c;
          }
          ex_bar();
          break;
        }
        run += rt;
        if (tid == 0) cd[3] = run;  // (not reached: the whole bucket's mass)
        ex_bar();
      }
      pick = cu[0];
      pm = cd[3];
      // broadcast to every CTA
      for (int g = 1; g < a.G; ++g)
        if (tid == 0) {
          ex_st64(ex_map(cu + 0, (uint32_t)g), pick);
          ex_st64(ex_map(cd + 3, (uint32_t)g), __double_as_longlong(pm));
        }
    }
    (void)level;
    ex_csync();
    pick = cu[0];
    pm = cd[3];
    *prefix_mass = pm;
    return pick;
  };

  // ---- top-k (count) cutoff, then W1 = mass of K1
  int bk = kNB0;
  if (topk) {
    double bf;
    find_bucket(false, 0.0, (uint64_t)rc.k, kNB0, &bk, &bf);
    const uint64_t need = (uint64_t)rc.k - (uint64_t)bf;
    double pmass;
    Ck = resolve(bk, 0, need, 0.0, 0.0, &pmass);
    // W1 = mass of the buckets before bk + the exact mass of bk's elements >= Ck
    double mb_bk;
    {
      int dummy_b;
      double dummy_before;
      (void)dummy_b;
      (void)dummy_before;
    }
    // mass before bucket bk (fixed order, from the per-thread values)
    if (tid == 0) cd[4] = 0.0;
    ex_bar();
    if (tid == bk / (kNB0 / kExThreads)) {
      double rr = mbefore;
      for (int j = 0; j < bk - tid * (kNB0 / kExThreads); ++j) rr += tm[j];
      cd[4] = rr;
    }
    ex_bar();
    mb_bk = cd[4];
    ex_bar();
    W1 = mb_bk + pmass;  // (pmass: the walk's mass of bk's first `need` elements, from 0)
  } else {
    W1 = mtot;
  }
  // ---- top-p cutoff over K1 (renormalised, R7; >= p W1, R8)
  if (rc.top_p < 1.0f) {
    const double target = (double)rc.top_p * W1;
    int bp;
    double bf;
    find_bucket(true, target, 0, topk ? bk + 1 : kNB0, &bp, &bf);
    if (bp < 0) bp = topk ? bk : kNB0 - 1;  // (rounding at the very top of the mass)
    double pmass;
    Cp = resolve(bp, 1, 0, bf, target, &pmass);
    if (topk && Cp < Ck) Cp = Ck;
  }
  // ---- min-p: the smallest binary32 z with exp((z - M)/tau) >= min_p (bisection on keys)
  if (rc.min_p > 0.0f) {
    if (tid == 0) {
      uint32_t lo = f2key(-INFINITY), hi = f2key(M);
      while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (exp(((double)key2f(mid) - (double)M) / (double)rc.tau) >= (double)rc.min_p) hi = mid;
        else lo = mid;
      }
      cu[1] = (uint64_t)hi << 32;  // every id with value >= key2f(hi)
    }
    ex_bar();
    Cm = cu[1];
    ex_bar();
  }
  uint64_t C3 = Ck > Cp ? Ck : Cp;
  C3 = Cm > C3 ? Cm : C3;

  // ---- the draw: W = mass of K3 in id order; per-CTA totals -> cluster prefix -> the CTA and the
  //      thread holding u*W walk their elements in id order
  double loc = 0.0;
  for_each([&](float z, int l) {
    if (make_comp(z, a.voff + l) >= C3) loc += weight(z);
  });
  const double ctot = ex_sum_d(loc, sd);
  if (tid == 0) ex_st64(ex_map(tots + rank, 0), __double_as_longlong(ctot));
  ex_csync();
  const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
  const double u = philox_uniform(seed, prm.request_id, a.step);
  if (rank == 0 && tid == 0) {
    double W = 0.0;
    for (int g = 0; g < a.G; ++g) W += tots[g];
    const double target = u * W;
    int gsel = -1;
    double pre = 0.0;
    for (int g = 0; g < a.G; ++g) {
      if (gsel < 0 && tots[g] > 0.0 && (pre + tots[g] > target)) gsel = g;
      if (gsel < 0) pre += tots[g];
    }
    int glast = -1;
    for (int g = 0; g < a.G; ++g)
      if (tots[g] > 0.0) glast = g;
    if (gsel < 0) {  // (u W at the top of the mass: the last kept id)
      gsel = glast;
      pre = 0.0;
      for (int g = 0; g < gsel; ++g) pre += tots[g];
    }
    for (int g = 0; g < a.G; ++g) {
      const uint32_t cg = ex_map(ctl + 8, (uint32_t)g);
      asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cg), "r"((uint32_t)gsel) : "memory");
      ex_st64(ex_map(cd + 8, (uint32_t)g), __double_as_longlong(target - pre));
      ex_st64(ex_map(cd + 9, (uint32_t)g), __double_as_longlong(W));
      ex_st64(ex_map(cd + 10, (uint32_t)g), __double_as_longlong(target >= pre + tots[gsel] ? 1.0 : 0.0));
    }
  }
  ex_csync();
  if ((int)rank == ctl[8]) {
    // this CTA holds the draw: walk its chunk in id order, rounds of 512 vectors (block scans)
    const double tgt = cd[8], W = cd[9];
    const bool at_top = cd[10] != 0.0;
    double run = 0.0;
    if (tid == 0) {
      ctl[9] = -1;   // found element (local id)
      ctl[11] = -1;  // last kept element (local id)
    }
    ex_bar();
    for (int base = v0; base < v1; base += kExThreads) {
      const int v = base + tid;
      float z[VEC];
      double wl[VEC];
      double vs = 0.0;
      int last = -1;
      if (v < v1) {
        R.vec(v, z);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          const bool kept = z[t] > -INFINITY && make_comp(z[t], a.voff + v * VEC + t) >= C3;
          wl[t] = kept ? weight(z[t]) : 0.0;
          vs += wl[t];
          if (kept) last = v * VEC + t;
        }
      } else {
#pragma unroll
        for (int t = 0; t < VEC; ++t) wl[t] = 0.0;
      }
      double rt;
      const double ex = ex_excl_scan_d(vs, &rt, sd) + run;
      if (!at_top && vs > 0.0 && ex <= tgt && tgt < ex + vs) {  // (one thread: the crossing vector)
        double c = ex;
        int pick = last;
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          c += wl[t];
          if (wl[t] > 0.0 && c > tgt) {
            pick = v * VEC + t;
            break;
          }
        }
        ctl[9] = pick;
      }
      if (last >= 0) atomicMax(&ctl[11], last);
      run += rt;
      ex_bar();
      if (ctl[9] >= 0) break;  // (uniform after the barrier)
    }
    if (tid == 0) {
      const int l = (ctl[9] >= 0) ? ctl[9] : ctl[11];  // (u W at the top of the mass: the last kept id)
      float zz[VEC];
      R.vec(l / VEC, zz);
      const float ztok = zz[l % VEC];
      const int tok = a.voff + l;
      const double wtok = exp(((double)ztok - (double)M) * inv_tau);
      const double lp = ((double)ztok - (double)M) * inv_tau - log(ri.S);
      a.ro.tokens[r] = tok;
      a.ro.logprobs[r] = (float)lp;
      if (a.ro.flogprobs) a.ro.flogprobs[r] = (float)log(wtok / W);
      if (a.ro.status) a.ro.status[r] = SAMPLER_ROW_OK;
      RowInfo o = ri;
      o.status = SAMPLER_ROW_OK;
      o.W = W;
      o.cutoff = C3;
      o.token = tok;
      a.ro.info[r] = o;
      ctl[12] = tok;
    }
    ex_bar();
    if (a.append && tid < 32) warp_append_token(a.hs, slot, ctl[12], tid);
  }
  ex_csync();  // no CTA leaves while another may still address its shared memory
}

// Debug: q[b, v] = final filtered distribution (w_v / W over K3; one-hot for greedy rows).
template <typename T>
__global__ void debug_q_kernel(const void* logits, int64_t ld, int V, int voff, int vloc,
                               const int32_t* slots, const sampling_params* params_dev,
                               const sampling_params* params_tab, int pen_mode, HistState hs,
                               const RowInfo* info, float* q) {
  const int r = blockIdx.y;
  const RowInfo ri = info[r];
  const int slot = row_slot(slots, r, hs.nslots, nullptr);
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

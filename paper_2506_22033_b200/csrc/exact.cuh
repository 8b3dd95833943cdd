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
  const uint64_t* step_dev;  // nullable: the decode step read on the device (sampler_set_step_source)
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
constexpr int kExOffWt = kExOffGat + kGat * 8;         // double [64] 2^(-j/64)
constexpr int kPmBlocks = 132;                         // presence-bitmap blocks (128 vectors) staged
constexpr int kExOffPm = kExOffWt + 64 * 8;            // u32 [kPmBlocks * 32] the chunk's bitmap
constexpr int kExOffScr = kExOffPm + kPmBlocks * 128;  // scratch: doubles / ints / u64
constexpr int kExOffKh = kExOffScr + 2048;             // bf16 rows: u16 counts per 16-bit value key [65536]
constexpr int kExactSmem = kExOffKh;                   // f32 rows
constexpr int kExactSmemBf16 = kExOffKh + 65536 * 2;   // bf16 rows
constexpr int kKhMaxChunk = 65535;                     // (u16 counts: chunks of at most this many elements)

#ifdef EXACT_PROF  // development timing marks (separate build: tools/exact_marks.sh)
__device__ uint64_t g_exprof[3][8][24];
#define EXPROF(i)                                                           \
  do {                                                                      \
    if (tid == 0 && r < 3) {                                                \
      uint64_t t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      g_exprof[r][rank][i] = t_;                                            \
      if (i == 15)                                                          \
        for (int j_ = 1; j_ < 24; ++j_)                                     \
          printf("EXPROF r%d c%d m%d %llu\n", r, (int)rank, j_,             \
                 (unsigned long long)g_exprof[r][rank][j_]);                \
    }                                                                       \
  } while (0)
#else
#define EXPROF(i) \
  do {            \
  } while (0)
#endif

#ifdef EXACT_STOP  // development: leave after stage i (timing of the stages; results invalid)
#define EXSTOP(i) \
  if (EXACT_STOP == i) return
#define EXACT_STOP_ON(i) (EXACT_STOP == i)
#else
#define EXSTOP(i)
#define EXACT_STOP_ON(i) false
#endif

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

// 2^x by the library (out of line: the rare far-tail / table paths; keeps the kernel's code small)
__device__ __noinline__ double ex_exp2(double x) { return exp2(x); }

// 2^-s for s in [0, ln2/64) via its series in s*ln2 (relative error < 3e-15)
__device__ __forceinline__ double exp2_neg_small(double d) {  // d = s * ln2 in [0, 0.0109)
  return 1.0 - d * (1.0 - d * (0.5 - d * (1.0 / 6.0 - d * (1.0 / 24.0 - d * (1.0 / 120.0)))));
}

// w = 2^-y = 2^(-b/64) * 2^-(y - b/64), b = floor(64 y): the bucket top from the 64-entry table
// 2^(-j/64) and an exact power of two, the rest by its short series; the far tail (y >= 32) by the
// library.  Out of line: called per element only off the hot loops (those use per-value tables).
__device__ __noinline__ double ex_weight(double y, const double* wtab) {
  const int b = (int)(y * 64.0);
  if (b >= kNB0 - 1) return exp2(-y);
  return wtab[b & 63] * __hiloint2double((1023 - (b >> 6)) << 20, 0) * exp2_neg_small((y - (double)b / 64.0) * kLn2);
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
  if (n <= 2 * kExThreads) {
    // small sets (the usual boundary bucket): rank sort of the distinct composites, one barrier
    // instead of the bitonic network's log2(N)^2 / 2 (45 at N = 512); in place via registers
    uint64_t x[2];
    int rk[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) x[q] = threadIdx.x + q * kExThreads < n ? buf[threadIdx.x + q * kExThreads] : 0ull;
    for (int j = 0; j < n; ++j) {
      const uint64_t y = buf[j];
      rk[0] += y > x[0] ? 1 : 0;
      rk[1] += y > x[1] ? 1 : 0;
    }
    ex_bar();
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (threadIdx.x + q * kExThreads < n) buf[rk[q]] = x[q];
    ex_bar();
    return;
  }
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

// order-preserving 16-bit key of a bf16 value (its bits) and back
__device__ __forceinline__ uint32_t okey_of_bits(uint32_t h) { return h ^ ((h & 0x8000u) ? 0xFFFFu : 0x8000u); }
__device__ __forceinline__ float val_of_okey(uint32_t k) {
  const uint32_t h = k ^ ((k & 0x8000u) ? 0x8000u : 0xFFFFu);
  return __uint_as_float(h << 16);
}

// the row as seen by one CTA: z' of local id l (penalties applied), element iteration by vectors
template <typename T>
struct ExRow {
  static constexpr int VEC = Dec<T>::N;
  const uint8_t* rowp;      // local slice of the row
  const uint32_t* pm;       // the slot's presence bitmap (phase A step-lane layout) from block kb
  int kb;
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
    const int k = (v >> 7) - kb, d = v & 127;
    return (pm[k * 32 + (d & 31)] >> ((d >> 5) * VEC)) & ((1u << VEC) - 1u);
  }
  __device__ __noinline__ float pen_value(int l) const {  // (rare: penalised elements only)
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
  __device__ __forceinline__ uint4 ld(int v) const { return *reinterpret_cast<const uint4*>(rowp + (int64_t)v * 16); }
  __device__ __forceinline__ void vec(int v, const uint4 u, float (&z)[Dec<T>::N]) const {
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
  double* wtab = reinterpret_cast<double*>(smem + kExOffWt);             // [64] 2^(-j/64)
  if (tid < 64) wtab[tid] = exp2(-(double)tid / 64.0);

  const int slot = row_slot(a.slots, r, a.hs.nslots, nullptr);  // (pending rows have a valid slot)
  const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
  const RowCfg rc = decode_row(prm, a.V, 1);
  const float M = ri.M;
  const double inv_tau = 1.0 / (double)rc.tau;
  const double l2e_tau = kLog2e / (double)rc.tau;

  ExRow<T> R;
  R.rowp = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * sizeof(T);
  R.pm = a.hs.pmask + (int64_t)slot * a.hs.spr * 32;
  R.kb = 0;
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
  {  // the chunk's presence bitmap into smem (one coalesced copy; every pass reads it per vector)
    const int kb = v0 >> 7, nb = v1 > v0 ? ((v1 - 1) >> 7) - kb + 1 : 0;
    if (nb <= kPmBlocks) {
      uint32_t* pms = reinterpret_cast<uint32_t*>(smem + kExOffPm);
      for (int i = tid; i < nb * 32; i += kExThreads) pms[i] = R.pm[(int64_t)kb * 32 + i];
      R.pm = pms;
      R.kb = kb;
    }
  }

  EXPROF(1);
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
  auto weight = [&](float z) -> double { return ex_weight(ycoord(z), wtab); };
  // one pass over the chunk's vectors (coalesced: vector v of thread tid, stride 512), the loads
  // of 4 vectors issued together (the passes are latency-bound otherwise)
  auto for_vecs = [&](auto&& fn) {
    constexpr int U = 4;
    for (int v = v0 + tid; v < v1; v += U * kExThreads) {
      uint4 u[U];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (v + j * kExThreads < v1) u[j] = R.ld(v + j * kExThreads);
      // (one copy of the body: the vectors picked by selects, not an unrolled loop - code size)
#pragma unroll 1
      for (int j = 0; j < U; ++j) {
        if (v + j * kExThreads >= v1) break;
        const uint4 uj = j == 0 ? u[0] : j == 1 ? u[1] : j == 2 ? u[2] : u[3];
        fn(v + j * kExThreads, uj);
      }
    }
  };
  auto for_each = [&](auto&& fn) {
    for_vecs([&](int v, const uint4 u) {
      float z[VEC];
      R.vec(v, u, z);
#pragma unroll
      for (int t = 0; t < VEC; ++t)
        if (z[t] > -INFINITY) fn(z[t], v * VEC + t);
    });
  };
  // bf16 rows (and the chunk's penalised ids in smem): pass 1 is an integer count histogram over the
  // 65 536 value keys; every float64 quantity is then computed once per distinct value (count x
  // weight), not per element.  (f32 rows, or more penalised ids than fit in smem: per element.)
  const bool keyed = (VEC == 8) && !R.ovf && (R.c1 - R.c0) <= kKhMaxChunk;
  uint32_t* kh = reinterpret_cast<uint32_t*>(smem + kExOffKh);  // [32768] pairs of u16 counts
  auto kcount = [&](uint32_t k) -> uint32_t { return (kh[k >> 1] >> ((k & 1u) * 16)) & 0xFFFFu; };
  // y and the level-0 bucket of a value (the same float64 arithmetic everywhere: consistent)
  auto bucket0 = [&](float z, double* yout) -> int {
    const double y = ycoord(z);
    *yout = y;
    if (!(y >= 0.0)) return -1;
    const double q = y * 64.0;
    return q >= (double)(kNB0 - 1) ? kNB0 - 1 : (int)q;
  };
  auto add_bucket = [&](float z, uint32_t c) {
    if (c == 0 || !(z > -INFINITY)) return;  // (-inf, NaN)
    double y;
    const int b = bucket0(z, &y);
    if (b < 0) return;
    const double rel = (b == kNB0 - 1) ? ex_exp2(-(y - (double)b / 64.0)) : exp2_neg_small((y - (double)b / 64.0) * kLn2);
    atomicAdd(&hcnt[b], c);
    smem_add_u64(&hmass[b], (uint64_t)c * (uint64_t)(rel * kFix40 + 0.5));
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
      const double rel = (b == nb - 1 && nb == kNB0) ? ex_exp2(-(y - ybase - (double)b / scale)) : exp2_neg_small(d);
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
    if (keyed && nb == kNB0) {
      // the bucket is a contiguous range of value keys (the bucket is monotone in the value):
      // its ends by bisection with the same float64 arithmetic, then an integer test per element
      // P(k) = bucket(k) > b and Q(k) = bucket(k) >= b are true-then-false over the keys from -max
      // (0x80) up: klo = first key with !P, khi = first key with !Q.  Two rounds of a 512-way search.
      {
        double y;
        const uint32_t ks = 0x80u + (uint32_t)tid * 128u;  // samples 0x80 + 128 t
        const int bs = bucket0(val_of_okey(ks), &y);
        const int np = __syncthreads_count(bs >= 0 && bs > b);   // samples with P (a prefix)
        const int nq = __syncthreads_count(bs >= 0 && bs >= b);  // samples with Q
        // the first !P key lies in (sample np-1, sample np]: threads 0..127 test its 128 keys
        const uint32_t pb0 = np > 0 ? 0x80u + (uint32_t)(np - 1) * 128u + 1u : 0x80u;
        const uint32_t qb0 = nq > 0 ? 0x80u + (uint32_t)(nq - 1) * 128u + 1u : 0x80u;
        const uint32_t kk = (tid < 128 ? pb0 : qb0) + (uint32_t)(tid & 127);
        const int bk2 = (tid < 256 && kk < 65536u) ? bucket0(val_of_okey(kk), &y) : -1;
        const bool pt = tid < 128 && kk < 65536u && bk2 >= 0 && bk2 > b;
        const bool qt = tid >= 128 && tid < 256 && kk < 65536u && bk2 >= 0 && bk2 >= b;
        const int cp = __syncthreads_count(pt), cq = __syncthreads_count(qt);
        if (tid == 0) {
          ctl[24] = (int)min(65536u, np > 0 ? pb0 + (uint32_t)cp : 0x80u);
          ctl[25] = (int)min(65536u, nq > 0 ? qb0 + (uint32_t)cq : 0x80u);
        }
        ex_bar();
      }
      const uint32_t klo = (uint32_t)ctl[24], khi = (uint32_t)ctl[25];  // keys [klo, khi)
      for_vecs([&](int v, const uint4 u) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        uint32_t hit = 0;  // elements of the vector in [klo, khi)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const uint32_t h = (t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu);
          hit |= (okey_of_bits(h) - klo < khi - klo ? 1u : 0u) << t;  // (unsigned range test)
        }
        if (!hit) return;
        hit &= ~R.pbits(v);  // (penalised: from the side list)
        while (hit) {
          const int t = __ffs(hit) - 1;
          hit &= hit - 1;
          const int l = v * 8 + t;
          if (l >= R.c1) break;
          const uint32_t h = (w[t >> 1] >> ((t & 1) * 16)) & 0xFFFFu;
          const uint32_t at = ex_atom_add(cnt_addr, 1u);
          if (at < (uint32_t)kGat) ex_st64(ex_map(gat + at, 0), make_comp(__uint_as_float(h << 16), a.voff + l));
        }
      });
      for (int e = tid; e < R.nside; e += kExThreads) {
        double y;
        const float z = side_z[e];
        if (z > -INFINITY && bucket0(z, &y) == b) {
          const uint32_t at = ex_atom_add(cnt_addr, 1u);
          if (at < (uint32_t)kGat) ex_st64(ex_map(gat + at, 0), make_comp(z, a.voff + side_id[e]));
        }
      }
      return;
    }
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
  EXPROF(2);
  EXSTOP(2);
  // ---- pass 1: level-0 histograms; the leader sums the cluster's and finds the cutoffs
  if (keyed) {
    for (int i = tid; i < 32768; i += kExThreads) kh[i] = 0;
    for (int i = tid; i < kNB0; i += kExThreads) {
      hcnt[i] = 0;
      hmass[i] = 0;
    }
    ex_bar();
    EXPROF(19);
    // every element of the chunk's whole vectors counted by its raw value key (one shared atomic
    // each, no per-element tests); then the penalised ones moved to their z' (side list) and the
    // ragged tail of the last chunk counted; -inf / NaN keys are skipped when the keys are read
    const int vfull = R.c1 / 8;
    for (int v = v0 + tid; v < vfull; v += 4 * kExThreads) {
      uint4 u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (v + j * kExThreads < vfull) u[j] = R.ld(v + j * kExThreads);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (v + j * kExThreads < vfull) {
          const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint32_t k = okey_of_bits((t & 1) ? (w[t >> 1] >> 16) : (w[t >> 1] & 0xFFFFu));
            atomicAdd(&kh[k >> 1], 1u << ((k & 1u) * 16));
          }
        }
    }
    if (tid < 8 && vfull * 8 + tid < R.c1) {  // the ragged tail (past the last whole vector)
      const uint32_t k = okey_of_bits(__float_as_uint(Dec<T>::load1(R.rowp, vfull * 8 + tid)) >> 16);
      atomicAdd(&kh[k >> 1], 1u << ((k & 1u) * 16));
    }
    ex_bar();
    for (int e = tid; e < R.nside; e += kExThreads) {  // penalised: out of the raw keys
      const uint32_t k = okey_of_bits(__float_as_uint(Dec<T>::load1(R.rowp, side_id[e])) >> 16);
      atomicSub(&kh[k >> 1], 1u << ((k & 1u) * 16));
    }
    ex_bar();
    EXPROF(20);
    for (int i = tid; i < 32768; i += kExThreads) {
      const uint32_t w = kh[i];
      if (!w) continue;
      add_bucket(val_of_okey(2u * i), w & 0xFFFFu);
      add_bucket(val_of_okey(2u * i + 1u), w >> 16);
    }
    for (int e = tid; e < R.nside; e += kExThreads) add_bucket(side_z[e], 1u);
    ex_bar();
  } else {
    histogram(0.0, 64.0, kNB0);
  }
  ex_csync();
  EXPROF(3);
  EXSTOP(3);
  // level-0 totals per bucket, in the leader; every CTA reads them (fixed order, deterministic)
  uint32_t tc[kNB0 / kExThreads];
  double tm[kNB0 / kExThreads];
  for (int j = 0; j < kNB0 / kExThreads; ++j) {
    const int b = tid * (kNB0 / kExThreads) + j;  // thread owns 4 consecutive buckets
    uint64_t m;
    tot_bucket(b, &tc[j], &m);
    tm[j] = (double)m * (1.0 / kFix40) * ex_exp2(-(double)b / 64.0);
  }
  ex_csync();  // (every CTA has read every histogram; they may be reused)
  EXPROF(4);
  EXSTOP(4);

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
  EXPROF(5);
    if (ctl[20] == 0 || rank != 0) {
      // (non-leaders only help gather)
    }
    int n = (int)ex_ld32(ex_map(ctl + 20, 0));
    ex_csync();
  EXPROF(6);
    int sbl = -1;  // the level-1 sub-bucket (level 1)
    if (n > kGat && b0 < kNB0 - 1) {  // too large: one more level inside bucket b0 (not the far tail)
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
        sm[j] = (double)m * (1.0 / kFix40) * ex_exp2(-(ybase + (double)b / scale));
      }
      ex_csync();
  EXPROF(7);
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
      sbl = sb;
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
  EXPROF(8);
    }
    if (n > kGat) {
      // near-ties: more than kGat elements in the level-1 sub-bucket (1/65536 octave of weight) or
      // in the far-tail bucket.  Radix rounds over the composite (z' desc, id asc) of the set's
      // elements: per round a 256-bin histogram of the next 8 bits (counts, masses relative to the
      // set's top weight in 2^-40 fixed point: the level's arithmetic), cluster totals, the bin
      // reaching the target; until it holds <= kGat elements, gathered and walked exactly below
      const bool lv1 = level == 1;
      const double yt = lv1 ? ybase + (double)sbl / scale : (double)b0 / 64.0;  // the set's top
      const double wtop = ex_exp2(-yt);
      auto member = [&](double y) -> bool {
        if (lv1) {
          const double q = (y - ybase) * scale;
          return q >= 0.0 && q < (double)kNB1 && (int)q == sbl;
        }
        return y * 64.0 >= (double)(kNB0 - 1);  // (level 0: the far-tail bucket b0 = kNB0 - 1)
      };
      auto relfix = [&](double y) -> uint64_t {
        const double rel = lv1 ? exp2_neg_small((y - yt) * kLn2) : ex_exp2(-(y - yt));
        return (uint64_t)(rel * kFix40 + 0.5);
      };
      uint32_t* tc2 = reinterpret_cast<uint32_t*>(gat);            // [256] cluster totals (scratch)
      uint64_t* tm2 = gat + 128;                                   // [256]
      if (tid == 0) {
        cu[4] = 0;          // klo
        cu[5] = ~0ull;      // khi
        cu[6] = 0;          // count above khi (in the sub-bucket)
        cu[7] = 0;          // fixed mass above khi
        ctl[26] = 56;       // shift
        ctl[27] = 0;        // done
      }
      ex_bar();
      for (;;) {
        const uint64_t klo = cu[4], khi = cu[5];
        const int sh = ctl[26];
        for (int i = tid; i < 256; i += kExThreads) {
          hcnt[i] = 0;
          hmass[i] = 0;
        }
        ex_csync();  // (every CTA's histogram is clear before any CTA adds to its own)
        for_each([&](float z, int l) {
          const double y = ycoord(z);
          if (!member(y)) return;
          const uint64_t c = make_comp(z, a.voff + l);
          if (c < klo || c > khi) return;
          const int bin = (int)((khi - c) >> sh);
          atomicAdd(&hcnt[bin], 1u);
          smem_add_u64(&hmass[bin], relfix(y));
        });
        ex_csync();
        for (int j = tid; j < 256; j += kExThreads) {
          uint32_t cj;
          uint64_t mj;
          tot_bucket(j, &cj, &mj);
          tc2[j] = cj;
          tm2[j] = mj;
        }
        ex_csync();  // (every remote histogram has been read)
        if (tid == 0) {
          uint64_t cb2 = cu[6], mb2 = cu[7];
          int js = -1, jl = -1;
          for (int j = 0; j < 256; ++j) {
            if (tc2[j] == 0) continue;
            jl = j;
            const bool hit = (mode == 0) ? (cb2 + tc2[j] >= need)
                                         : (before + (double)(mb2 + tm2[j]) * (1.0 / kFix40) * wtop >= target);
            if (hit) {
              js = j;
              break;
            }
            cb2 += tc2[j];
            mb2 += tm2[j];
          }
          if (js < 0) {  // (rounding shortfall: the last non-empty bin)
            js = jl;
            cb2 -= tc2[jl];
            mb2 -= tm2[jl];
          }
          const uint64_t nhi = khi - ((uint64_t)js << sh);
          const uint64_t span = (sh >= 64) ? ~0ull : ((1ull << sh) - 1ull);
          cu[4] = (nhi - klo > span) ? nhi - span : klo;
          cu[5] = nhi;
          cu[6] = cb2;
          cu[7] = mb2;
          ctl[27] = (tc2[js] <= (uint32_t)kGat || sh == 0) ? 1 : 0;
          ctl[26] = sh - 8;
        }
        ex_bar();
        if (ctl[27]) break;
      }
      // the elements of the final interval into the leader's buffer
      const uint64_t klo = cu[4], khi = cu[5];
      if (tid == 0) ctl[20] = 0;
      ex_csync();
      const uint32_t cnt_addr = ex_map(ctl + 20, 0);
      for_each([&](float z, int l) {
        if (!member(ycoord(z))) return;
        const uint64_t c = make_comp(z, a.voff + l);
        if (c < klo || c > khi) return;
        const uint32_t at = ex_atom_add(cnt_addr, 1u);
        if (at < (uint32_t)kGat) ex_st64(ex_map(gat + at, 0), c);
      });
      ex_csync();
      n = (int)ex_ld32(ex_map(ctl + 20, 0));
      if (mode == 0) need -= cu[6];                       // (count from the interval's start)
      before += (double)cu[7] * (1.0 / kFix40) * wtop;    // (the walk's mass from the interval's start)
      ex_csync();
    }
    n = min(n, kGat);  // (the refinement above leaves at most kGat)
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
  EXPROF(9);
    pick = cu[0];
    pm = cd[3];
    *prefix_mass = pm;
    return pick;
  };

  // ---- top-k (count) cutoff, then W1 = mass of K1
  EXPROF(10);
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
  EXPROF(11);
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
  EXPROF(12);
  EXSTOP(12);
  //      thread holding u*W walk their elements in id order.  Every CTA: the kept mass of its chunk in
  //      rounds of 512 vectors (id order), per (round, warp) into smem; the CTA totals from those.
  // bf16 rows: the weights of the values with exponent in [2^-16, 2^8) from a table (one entry per
  // value, the same float64 arithmetic as weight(); built over the key histogram, no longer needed)
  constexpr int kE0 = 127 - 16, kNE = 24;
  double* wk = reinterpret_cast<double*>(smem + kExOffKh);  // [2][kNE][128]
  double* side_w = wk + 2 * kNE * 128;  // [kSide] weights of the side list's z'
  // the side-list index of each vector's first penalised element (prefix of the bitmap counts)
  uint16_t* prank = reinterpret_cast<uint16_t*>(side_w + kSide);  // [chunk vectors <= 8192]
  static_assert((2 * kNE * 128 + kSide) * 8 + 8192 * 2 <= 65536 * 2, "tables overlay the key histogram");
  if (keyed) {
    for (int e = tid; e < R.nside; e += kExThreads) side_w[e] = side_z[e] > -INFINITY ? weight(side_z[e]) : 0.0;
    {
      const int S2 = (v1 - v0 + kExThreads - 1) / kExThreads;
      const int a0 = min(v1, v0 + tid * S2), a1 = min(v1, a0 + S2);
      int cnt = 0;
      for (int v = a0; v < a1; ++v) cnt += __popc(R.pbits(v));
      const int lane = tid & 31, w = tid >> 5;
      const int incl = warp_incl_scan_i(cnt, lane);
      if (lane == 31) si[w] = incl;
      ex_bar();
      int run = incl - cnt;
      for (int i = 0; i < w; ++i) run += si[i];
      for (int v = a0; v < a1; ++v) {
        prank[v - v0] = (uint16_t)run;
        run += __popc(R.pbits(v));
      }
    }
    for (int i = tid; i < 2 * kNE * 128; i += kExThreads) {
      const uint32_t h = ((uint32_t)(i / (kNE * 128)) << 15) | ((uint32_t)(kE0 + (i / 128) % kNE) << 7) | (uint32_t)(i & 127);
      const float z = __uint_as_float(h << 16);
      wk[i] = (z <= M) ? weight(z) : 0.0;
    }
    ex_bar();
  }
  EXPROF(21);
  if (EXACT_STOP_ON(21)) return;
  const uint32_t id3c = (uint32_t)comp_id(C3);
  // bf16 kept test in the 16-bit value-key order: kept <=> kb3 + [local id > l3] <= okey <= okey(+max)
  // (ties at the cutoff value kept up to its id; a cutoff value that is no bf16 value has no ties)
  int kb3 = 0x80;                 // (no cutoff: every finite value, from okey(-max))
  int64_t l3 = INT64_MAX;
  if (keyed && C3 != 0) {
    const float v3 = comp_val(C3);
    const uint32_t b3 = __float_as_uint(v3);
    if ((b3 & 0xFFFFu) == 0u) {  // a bf16 value: +0 stands for both zeros (composite order)
      kb3 = (int)okey_of_bits(b3 >> 16);
      l3 = (int64_t)id3c - a.voff;
    } else {                     // the first value key above v3 (bisection, one thread)
      if (tid == 0) {
        uint32_t lo = 0x80u, hi = 0xFF80u;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (val_of_okey(mid) > v3) hi = mid;
          else lo = mid + 1;
        }
        ctl[16] = (int)lo;
      }
      ex_bar();
      kb3 = ctl[16];
    }
  }
  // the kept weights w[0..VEC) of vector v (0 if not kept); *lastk = its last kept local id
  auto vec_w = [&](int v, const uint4 u, double* w, int* lastk) {
    const int lb = v * VEC;
    const uint32_t pb = R.pbits(v);
    if (VEC == 8 && keyed) {
      // unpenalised elements: the kept test on the value key, the weight from the per-value table
      // (values outside it after, rarely); penalised ones from the side list (weights precomputed)
      const uint32_t ok = ~pb & (lb + 8 <= R.c1 ? 0xFFu : (1u << max(0, R.c1 - lb)) - 1u);
      uint32_t kept_m = 0, slow = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const uint32_t wd = t < 2 ? u.x : t < 4 ? u.y : t < 6 ? u.z : u.w;
        uint32_t h = (t & 1) ? (wd >> 16) : (wd & 0xFFFFu);
        h = h == 0x8000u ? 0u : h;  // (-0 is +0)
        const uint32_t k = okey_of_bits(h);
        const uint32_t kt = (uint32_t)kb3 + ((int64_t)(lb + t) > l3 ? 1u : 0u);
        const bool kept = ((ok >> t) & 1u) && k >= kt && k <= 0xFF7Fu;  // (finite, at or above the cutoff)
        const uint32_t wi = (h & 0x7FFFu) - (uint32_t)(kE0 << 7);  // index within the sign's table
        const bool inw = wi < (uint32_t)(kNE * 128);
        const double wt = wk[inw ? wi + (h >> 15) * (kNE * 128) : 0u];
        w[t] = (kept && inw) ? wt : 0.0;
        kept_m |= (kept ? 1u : 0u) << t;
        slow |= (kept && !inw ? 1u : 0u) << t;
      }
      if (slow) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if ((slow >> t) & 1u) {
            const uint32_t wd = t < 2 ? u.x : t < 4 ? u.y : t < 6 ? u.z : u.w;
            const uint32_t h = (t & 1) ? (wd >> 16) : (wd & 0xFFFFu);
            w[t] = weight(__uint_as_float(h << 16));
          }
      }
      const uint32_t pq = pb & (lb + 8 <= R.c1 ? 0xFFu : (1u << max(0, R.c1 - lb)) - 1u);
      if (pq) {
        int e = prank[v - v0];  // its first penalised element's side entry (then consecutive)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if ((pq >> t) & 1u) {
            const float z = side_z[e];
            const bool kept = z > -INFINITY && make_comp(z, a.voff + lb + t) >= C3;
            w[t] = kept ? side_w[e] : 0.0;
            kept_m |= (kept ? 1u : 0u) << t;
            ++e;
          }
      }
      if (kept_m) *lastk = lb + 31 - __clz(kept_m);
      return;
    }
    float z[VEC];
    R.vec(v, u, z);
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      const bool kept = z[t] > -INFINITY && make_comp(z[t], a.voff + lb + t) >= C3;
      w[t] = kept ? weight(z[t]) : 0.0;
      *lastk = kept ? lb + t : *lastk;
    }
  };
  // rounds of 512 vectors in id order (vector v0 + 512 i + tid: coalesced, loads of 4 rounds in
  // flight): per round the warps' kept masses (fixed-order warp sums) into smem; then the round,
  // the warp and the lane holding the target, each from those sums (no per-round block barrier)
  const int nr = (v1 - v0 + kExThreads - 1) / kExThreads;  // rounds (<= kGat / kExW)
  double* rs = reinterpret_cast<double*>(gat);              // [nr][kExW] (the gather list is done)
  const int lane = tid & 31, wp = tid >> 5;
  int last = -1;
  uint4 un[4];  // (the next 4 rounds' vectors in flight while 4 are processed)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int v = v0 + j * kExThreads + tid;
    if (j < nr && v < v1) un[j] = R.ld(v);
  }
  for (int i0 = 0; i0 < nr; i0 += 4) {
    uint4 u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u[j] = un[j];
      const int v = v0 + (i0 + 4 + j) * kExThreads + tid;
      if (i0 + 4 + j < nr && v < v1) un[j] = R.ld(v);
    }
#pragma unroll 1
    for (int j = 0; j < 4 && i0 + j < nr; ++j) {
      const int v = v0 + (i0 + j) * kExThreads + tid;
      const uint4 uj = j == 0 ? u[0] : j == 1 ? u[1] : j == 2 ? u[2] : u[3];
      double w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#if defined(EXACT_EXP) && EXACT_EXP == 3
      w[0] = (double)uj.x;
#else
      if (v < v1) vec_w(v, uj, w, &last);
#endif
      double ls = 0.0;
#pragma unroll
      for (int q = 0; q < VEC; ++q) ls += w[q];
#if !(defined(EXACT_EXP) && EXACT_EXP == 2)
      ls = warp_sum_d(ls);
#endif
      if (lane == 0) rs[(i0 + j) * kExW + wp] = ls;
    }
  }
  if (tid == 0) ctl[11] = -1;  // last kept element (local id)
  ex_bar();
  if (last >= 0) atomicMax(&ctl[11], last);
  // the CTA total: round totals (warps in order), scanned 32 rounds at a time (the same arithmetic
  // as the search below, so that the two agree to the bit)
  if (tid < 32) {
    double run = 0.0;
    for (int i0 = 0; i0 < nr; i0 += 32) {
      const int i = i0 + lane;
      double tot = 0.0;
      if (i < nr)
        for (int k = 0; k < kExW; ++k) tot += rs[i * kExW + k];
      run += __shfl_sync(0xFFFFFFFFu, warp_incl_scan_d(tot, lane), 31);
    }
    if (lane == 0) ex_st64(ex_map(tots + rank, 0), __double_as_longlong(run));
  }
  ex_csync();
  EXPROF(13);
  EXSTOP(13);
  const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
  const double u = philox_uniform(seed, prm.request_id, a.step_dev ? *a.step_dev : a.step);
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
  EXPROF(14);
  EXSTOP(14);
  if ((int)rank == ctl[8]) {
    // this CTA holds the draw: the round, the warp and the lane holding the target from its sums
    const double tgt = cd[8], W = cd[9];
    const bool at_top = cd[10] != 0.0;
    if (tid == 0) ctl[9] = -1;  // found element (local id)
    EXPROF(16);
    if (EXACT_STOP_ON(16)) return;
    ex_bar();
    EXPROF(17);
    // warp 0: round totals (warps in order), their prefix; the round rr holding the target and the
    // mass before it, then the warp ww inside it
    if (tid < 32) {
      double run = 0.0;
      int rr = -1, ww = -1;
      double before = 0.0;
      for (int i0 = 0; i0 < nr && rr < 0; i0 += 32) {
        const int i = i0 + lane;
        double tot = 0.0;
        if (i < nr)
          for (int k = 0; k < kExW; ++k) tot += rs[i * kExW + k];
        const double incl = warp_incl_scan_d(tot, lane);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, i < nr && tot > 0.0 && run + incl > tgt);
        if (bal) {
          const int src = __ffs(bal) - 1;
          rr = i0 + src;
          before = __shfl_sync(0xFFFFFFFFu, run + incl - tot, src);
        }
        run += __shfl_sync(0xFFFFFFFFu, incl, 31);
      }
      if (rr >= 0 && !at_top) {
        const double wv = lane < kExW ? rs[rr * kExW + lane] : 0.0;
        const double incl = warp_incl_scan_d(wv, lane);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, lane < kExW && wv > 0.0 && before + incl > tgt);
        const int src = bal ? __ffs(bal) - 1 : -1;
        ww = src;
        if (src >= 0) before = __shfl_sync(0xFFFFFFFFu, before + incl - wv, src);
      }
      if (lane == 0) {
        ctl[14] = rr;
        ctl[15] = ww;
        cd[11] = before;
      }
    }
    ex_bar();
    {
      const int rr = ctl[14], ww = ctl[15];
      if (rr >= 0 && ww >= 0 && wp == ww) {
        // the warp holding the target: its lanes' vectors again, a warp scan, the crossing lane
        // walks its elements in order
        const int v = v0 + rr * kExThreads + tid;
        double w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int lk = -1;
        if (v < v1) vec_w(v, R.ld(v), w, &lk);
        double ls = 0.0;
#pragma unroll
        for (int q = 0; q < VEC; ++q) ls += w[q];
        const double incl = warp_incl_scan_d(ls, lane);
        const double before = cd[11];
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, ls > 0.0 && before + incl > tgt);
        int lmax = lk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xFFFFFFFFu, lmax, o));
        if (bal) {
          if (lane == __ffs(bal) - 1) {
            double c = before + incl - ls;
            int p = lk;  // (rounding inside the lane: its last kept)
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
              c += w[q];
              if (w[q] > 0.0 && c > tgt) {
                p = v * VEC + q;
                break;
              }
            }
            ctl[9] = p;
          }
        } else if (lane == 0) {
          ctl[9] = lmax;  // (rounding: the target at the warp's very top - its last kept id)
        }
      }
    }
    ex_bar();
    EXPROF(18);
    if (tid == 0) {
      const int l = (ctl[9] >= 0) ? ctl[9] : ctl[11];  // (u W at the top of the mass: the last kept id)
      float zz[VEC];
      R.vec(l / VEC, R.ld(l / VEC), zz);
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
  EXPROF(15);
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

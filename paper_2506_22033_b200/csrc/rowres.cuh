// rowres.cuh — the sampling step as one persistent cluster kernel with the rows resident in
// distributed shared memory (DSMEM).
//
// The batch [B x V] is cut by rows: a thread-block cluster of C CTAs takes one row at a time, CTA c
// holding the row's vocabulary chunk [c*Lc, (c+1)*Lc) in its shared memory (1-D bulk copies, TMA
// engine).  Every pass of the row then runs from shared memory, and the row crosses HBM exactly
// once (the logits z_s of the last stage).  Per CTA and row (one "row group" of 4 warps):
//   pen     the penalised ids of the chunk (presence bitmap + the slot's unique-token entries of
//           the chunk, located by the per-slot prefix table) get their exact penalised value
//           z' = ApplyPenalty(z, y_<s) (R1-R3); in the chunk they
//           are masked to -inf, so the bulk passes below see only unpenalised logits;
//   A1      max over the chunk (NaN-propagating: NaN / +inf rows are detected for free) and one
//           max per thread;  T_c = the keff-th largest thread max (keff = top-k, or 1 for greedy):
//           keff distinct elements are >= T_c, so every element of the row's top-k in this chunk
//           is >= T_c;
//   A2      S_c = sum 2^((z' - m_c) log2(e)/tau) (P:149's softmax denominator, relative to the
//           chunk max m_c: every term <= 1, no rebasing), and every element >= T_c pushed
//           straight into the leader CTA's candidate list (DSMEM stores);
//   send    the chunk record {m_c, S_c, frontier, count} to the row's leader, CTA (row index mod C),
//           one remote mbarrier arrive.
// The leader's decider warp merges the C records (M = max m_c, S = sum S_c 2^((m_c - M) c),
// frontier = max, candidates >= frontier), takes the exact top-k by (z' desc, id asc), and runs the
// decision of merge.cuh (top-k -> top-p -> min-p in float64, Philox draw in id order, logprobs,
// history append) while the row groups already stream the next rows: a row's decision overlaps
// the streaming of the C-1 rows after it.  Two row groups per CTA, each with its own buffer, keep
// two rows in flight per SM (one group's latency-bound steps overlap the other's passes).
// Rows whose kept set is not bounded by the candidates (top-p / min-p-only, unfiltered, top_k >
// K_cand) leave a pending RowInfo {M, S} for exact.cuh.  Mode 1 (vocab-sharded phase 1) writes the
// row's candidate record instead of deciding.
#pragma once
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "philox.cuh"

namespace smp {

constexpr int kRNB = 2;                      // chunk buffers per CTA
constexpr int kSW = 12;                      // stream warps (the pass over each chunk)
constexpr int kST = kSW * 32;                // stream threads
constexpr int kNF = 2;                       // finisher groups (rows alternate between them)
constexpr int kFW = 4;                       // warps per finisher group
constexpr int kFT = kFW * 32;                // threads per finisher group
constexpr int kNS = 3;                       // summary slots (rows passed, not yet finished)
constexpr int kRProdW = kSW + kNF * kFW;     // producer warp index
constexpr int kRDecW = kRProdW + 1;          // decider warp index
constexpr int kRThreads = (kRDecW + 1) * 32;
constexpr int kPT = 4;                       // penalised ids staged per stream thread and row
constexpr int kPenS = 256;                   // penalised (id, z') entries per summary slot (more: slow path)
constexpr int kRCMax = 16;                   // max cluster size
constexpr int kRCapL = 256;                  // local candidate list per finisher group
constexpr int kLcAlign = 128;                // chunk length granularity (16-byte bitmap rows, 16-byte copies)

// per-row staging, written by the producer next to the bulk copies of the chunk
struct __align__(16) RowStage {
  sampling_params prm;
  int32_t slot, pad[3];
};

// chunk record sent to the row's leader
struct __align__(16) RecC {
  float m;          // max z' over the chunk
  uint32_t flags;   // bit0 NaN / +inf seen
  double s;         // sum 2^((z' - m) * c)
  uint64_t front;   // every element of the chunk with composite >= front is in the list (0: all)
  uint64_t best;    // greedy rows: the chunk's best composite
  int32_t n;        // list entries
  int32_t pad[3];
};

struct RArgs {
  const void* logits;
  int64_t ld;
  int B, V, voff, vloc;
  int C;        // cluster size
  int Lc;       // chunk length (elements, multiple of kLcAlign)
  int cap;      // sorted candidate list capacity per chunk in the leader (>= max_top_k)
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  int kcand, pen_mode, mode, append;
  HistState hs;
  RowOut ro;
  uint8_t* out_records;
  int64_t out_stride;
  uint64_t* trace;  // SMP_TRACE builds only (development): [CTA][kTrRows][16] globaltimer stamps
};

// Development timeline (tools/trace_row.py): compiled in only with -DSMP_TRACE, never in the
// product library.  Slot = (CTA, row of the cluster < kTrRows, event < 16).
constexpr int kTrRows = 64;
#ifdef SMP_TRACE
#define RTR(it, ev)                                                                                   \
  do {                                                                                                \
    if (a.trace && (it) < kTrRows) a.trace[((int64_t)blockIdx.x * kTrRows + (it)) * 16 + (ev)] = gtimer(); \
  } while (0)
#define RTV(it, ev, val)                                                                               \
  do {                                                                                                  \
    if (a.trace && (it) < kTrRows) a.trace[((int64_t)blockIdx.x * kTrRows + (it)) * 16 + (ev)] = (uint64_t)(val); \
  } while (0)
#else
#define RTV(it, ev, val) \
  do {                   \
  } while (0)
#define RTR(it, ev) \
  do {              \
  } while (0)
#endif

// ---- shared-memory layout (host and device) ----------------------------------------
// summary slot (one passed row): per stream thread t its max (incl. penalised), exp-sum reference and
// sum; per group (2 vectors of one thread) its max key; the penalised (id, z') of the chunk; flags
struct SlotHdr {
  sampling_params prm;
  int32_t slot, npen, bad, pad;
};
__host__ __device__ inline int slot_bytes(int Lc, int esz) {
  const int keys = (Lc / 16) * (esz == 2 ? 2 : 4);
  return (int)sizeof(SlotHdr) + kST * 12 + (keys + 15) / 16 * 16 + kPenS * 8;
}
struct RLay {
  int buf, bm, stg, pme, sl, slb, rinfo, hdr, rec, pool, top, wv, byid, dscr, fscr, bslot, bar, total;
};
constexpr int kFScrBytes = kRCapL * 8 + 256;
__host__ __device__ inline RLay rlayout(int C, int Lc, int esz, int cap) {
  RLay l;
  int o = 0;
  auto A = [&o](int bytes) {
    const int r = o;
    o += (bytes + 127) / 128 * 128;
    return r;
  };
  l.buf = A(kRNB * Lc * esz);
  l.bm = A(kRNB * (Lc / 8));
  l.stg = A(kRNB * (int)sizeof(RowStage));
  l.pme = A(kST * kPT * 4);
  l.slb = (slot_bytes(Lc, esz) + 127) / 128 * 128;
  l.sl = A(kNS * l.slb);
  l.rinfo = A((int)sizeof(RowStage));
  l.hdr = A(C * (int)sizeof(RecC));
  l.rec = A(C * cap * 8);
  l.pool = A(C * cap * 8);
  l.top = A(SAMPLER_KCAND_MAX * 8);
  l.wv = A((SAMPLER_KCAND_MAX + 64) * 8);  // (also warp_topk's survivor scratch)
  l.byid = A(SAMPLER_KCAND_MAX * 8);
  l.dscr = A(512);
  l.fscr = A(kNF * kFScrBytes);
  l.bslot = A(kNF * 2 * kRCMax * 4);  // row bounds exchanged between the cluster's CTAs
  l.bar = A((2 * kRNB + 2 * kNS + kNF + 1 + kRCMax) * 8);
  l.total = o;
  return l;
}

// ---- cluster / DSMEM PTX ------------------------------------------------------------
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_num() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_st64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void cl_st128(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void cl_fence() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
// arrive (count 1) on an mbarrier of another CTA of the cluster; releases this thread's prior writes
__device__ __forceinline__ void cl_arrive_remote(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
// wait on a local mbarrier whose arrivals may come from other CTAs (cluster-scope acquire)
// (back-off between polls: a waiting warp must not take issue slots from the row groups)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(SMP_SLEEP_NS);
  }
}
// 4-byte asynchronous global -> shared copy (LDGSTS): gathers that complete behind other work
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// named barrier of one finisher group (ids 1..kNF)
__device__ __forceinline__ void fbar(int f) { asm volatile("bar.sync %0, %1;" ::"r"(f + 1), "n"(kFT) : "memory"); }

// ---- element formats ----------------------------------------------------------------
template <typename T>
struct RV;
template <>
struct RV<__nv_bfloat16> {
  static constexpr int N = 8;
  // bit t of b set => element t becomes -inf
  static __device__ __forceinline__ uint4 mask(uint4 u, uint32_t b) {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if ((b >> (2 * i)) & 1u) w[i] = (w[i] & 0xFFFF0000u) | 0xFF80u;
      if ((b >> (2 * i + 1)) & 1u) w[i] = (w[i] & 0x0000FFFFu) | 0xFF800000u;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  static __device__ __forceinline__ __nv_bfloat162 h2(uint32_t w) { return *reinterpret_cast<__nv_bfloat162*>(&w); }
  // NaN-propagating max of the 8 elements, as a bf16x2 pair
  static __device__ __forceinline__ __nv_bfloat162 vmax2_nan(uint4 u) {
    return __hmax2_nan(__hmax2_nan(h2(u.x), h2(u.y)), __hmax2_nan(h2(u.z), h2(u.w)));
  }
  static __device__ __forceinline__ float vmax(uint4 u) {
    const __nv_bfloat162 m = __hmax2(__hmax2(h2(u.x), h2(u.y)), __hmax2(h2(u.z), h2(u.w)));
    return fmaxf(__low2float(m), __high2float(m));
  }
  static __device__ __forceinline__ float elem(uint4 u, int t) {
    const uint32_t w = (t < 2) ? u.x : (t < 4) ? u.y : (t < 6) ? u.z : u.w;
    return __uint_as_float((t & 1) ? (w & 0xFFFF0000u) : (w << 16));
  }
  static __device__ __forceinline__ float at(const uint8_t* buf, int i) {
    return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(buf)[i] << 16);
  }
  // sum over the 8 elements of 2^((z - m) * c): exact bf16 -> f32 differences (FFMA with a bf16
  // operand), packed multiply, MUFU ex2, packed adds; masked (-inf) elements give 0
  static __device__ __forceinline__ float esum(uint4 u, float nm, float, uint64_t c2) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint64_t p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float a, b;
      asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
          "fma.rn.f32.bf16 %0, l, %3, %4;\n\tfma.rn.f32.bf16 %1, h, %3, %4;}"
          : "=f"(a), "=f"(b)
          : "r"(w[i]), "h"((unsigned short)0x3F80), "f"(nm));
      uint64_t t2, x2;
      asm("mov.b64 %0, {%1, %2};" : "=l"(t2) : "f"(a), "f"(b));
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(x2) : "l"(t2), "l"(c2));
      float xa, xb;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(xa), "=f"(xb) : "l"(x2));
      const float ea = ex2f(xa), eb = ex2f(xb);
      asm("mov.b64 %0, {%1, %2};" : "=l"(p[i]) : "f"(ea), "f"(eb));
    }
    uint64_t s01, s23, s;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s01) : "l"(p[0]), "l"(p[1]));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s23) : "l"(p[2]), "l"(p[3]));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(s01), "l"(s23));
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(s));
    return a + b;
  }
};
template <>
struct RV<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ uint4 mask(uint4 u, uint32_t b) {
    if (b & 1u) u.x = 0xFF800000u;
    if (b & 2u) u.y = 0xFF800000u;
    if (b & 4u) u.z = 0xFF800000u;
    if (b & 8u) u.w = 0xFF800000u;
    return u;
  }
  static __device__ __forceinline__ float vmax_nan(uint4 u) {
    return fmax_nan(fmax_nan(__uint_as_float(u.x), __uint_as_float(u.y)),
                    fmax_nan(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  static __device__ __forceinline__ float vmax(uint4 u) {
    return fmaxf(fmaxf(__uint_as_float(u.x), __uint_as_float(u.y)), fmaxf(__uint_as_float(u.z), __uint_as_float(u.w)));
  }
  static __device__ __forceinline__ float elem(uint4 u, int t) {
    return __uint_as_float(t == 0 ? u.x : t == 1 ? u.y : t == 2 ? u.z : u.w);
  }
  static __device__ __forceinline__ float at(const uint8_t* buf, int i) {
    return reinterpret_cast<const float*>(buf)[i];
  }
  static __device__ __forceinline__ float esum(uint4 u, float nm, float cf, uint64_t) {
    const float z[4] = {__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w)};
    float e[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) e[i] = ex2f(__fmul_rn(__fadd_rn(z[i], nm), cf));
    return (e[0] + e[1]) + (e[2] + e[3]);
  }
};

// bitmap bits of vector v (VEC elements) from the chunk bitmap (bit i = element i)
template <int VEC>
__device__ __forceinline__ uint32_t vec_bits(const uint8_t* bm, int v) {
  if (VEC == 8) return bm[v];
  return (bm[v >> 1] >> ((v & 1) * 4)) & 0xFu;
}

// The keff largest of pool[0..n) (unique composites) into top[0..min(n, keff)), sorted descending;
// one warp.  The keff-th largest value key by bitwise radix select (ballot counts; the bits above
// the first one where the largest and smallest key differ are common to all), the survivors (key
// above it, and the ties at it) compacted into scr (>= SAMPLER_KCAND_MAX + 64 entries, else the
// id part is selected too), then a rank sort of the survivors.
__device__ __forceinline__ int warp_topk(const uint64_t* pool, int n, int keff, uint64_t* scr, uint64_t* top,
                                         int lane) {
  uint64_t kc = 0;  // survivors: composites >= kc
  if (n > keff) {
    uint32_t kmax = 0, kmin = 0xFFFFFFFFu;
    for (int i = lane; i < n; i += 32) {
      const uint32_t h = (uint32_t)(pool[i] >> 32);
      kmax = max(kmax, h);
      kmin = min(kmin, h);
    }
    kmax = __reduce_max_sync(kFull, kmax);
    kmin = __reduce_min_sync(kFull, kmin);
    const int top_bit = 31 - __clz(kmax ^ kmin);  // (-1: all keys equal)
    uint32_t hk = top_bit >= 0 ? (kmax & ~((2u << top_bit) - 1u)) : kmax;
#pragma unroll 1
    for (int b = top_bit; b >= 0; --b) {
      const uint32_t cand = hk | (1u << b);
      uint32_t c = 0;
      for (int i = lane; i < n; i += 32) c += ((uint32_t)(pool[i] >> 32) >= cand) ? 1u : 0u;
      if ((int)__reduce_add_sync(kFull, c) >= keff) hk = cand;
    }
    kc = (uint64_t)hk << 32;
    uint32_t ge = 0;
    for (int i = lane; i < n; i += 32) ge += ((uint32_t)(pool[i] >> 32) >= hk) ? 1u : 0u;
    if ((int)__reduce_add_sync(kFull, ge) > SAMPLER_KCAND_MAX + 64) {  // massive ties at hk: the id part too
      uint32_t gt = 0;
      for (int i = lane; i < n; i += 32) gt += ((uint32_t)(pool[i] >> 32) > hk) ? 1u : 0u;
      const int need = keff - (int)__reduce_add_sync(kFull, gt);
      uint32_t lk = 0;
#pragma unroll 1
      for (int b = 31; b >= 0; --b) {
        const uint32_t cand = lk | (1u << b);
        uint32_t c = 0;
        for (int i = lane; i < n; i += 32)
          c += ((uint32_t)(pool[i] >> 32) == hk && (uint32_t)pool[i] >= cand) ? 1u : 0u;
        if ((int)__reduce_add_sync(kFull, c) >= need) lk = cand;
      }
      kc |= lk;
    }
  }
  int m = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t v = (i < n) ? pool[i] : 0ull;
    const bool keep = i < n && v >= kc;
    const unsigned bal = __ballot_sync(kFull, keep);
    if (keep) scr[m + __popc(bal & ((1u << lane) - 1u))] = v;
    m += __popc(bal);
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) {
    const uint64_t c = scr[i];
    int rk = 0;
    for (int j = 0; j < m; ++j) rk += (scr[j] > c) ? 1 : 0;
    if (rk < keff) top[rk] = c;
  }
  __syncwarp();
  return min(m, keff);
}

template <typename T>
__global__ void __launch_bounds__(kRThreads, 1) row_kernel(const __grid_constant__ RArgs a) {
  constexpr int VEC = RV<T>::N;
  constexpr int ESZ = (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  const RLay L = rlayout(a.C, a.Lc, ESZ, a.cap);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cl_rank(), q = cl_id(), nclus = cl_num();
  const int C = a.C;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* full = bar;                  // [kRNB] chunk landed
  uint64_t* empty = full + kRNB;         // [kRNB] chunk consumed by the stream warps
  uint64_t* spass = empty + kRNB;        // [kNS] summary slot written (stream warps)
  uint64_t* sfree = spass + kNS;         // [kNS] summary slot released (finisher)
  uint64_t* bound = sfree + kNS;         // [kNF] the C chunk bounds of the finisher's current row
  uint64_t* recfull = bound + kNF;       // [1] the C chunk records of a row this CTA leads
  uint64_t* slotfree = recfull + 1;      // [kRCMax] leader l has consumed our last list
  const int nrows = (a.B > (int)q) ? (a.B - (int)q + (int)nclus - 1) / (int)nclus : 0;  // rows of this cluster
  const int c0 = (int)rank * a.Lc;                                // first local id of this CTA's chunk
  const int nval = max(0, min(a.Lc, a.vloc - c0));                // valid elements of the chunk
  const int nvec = (nval + VEC - 1) / VEC;
  const int nfull = nval / VEC;                                   // vectors without a ragged tail
  const uint32_t tailmask = (nvec > nfull) ? (~((1u << (nval - nfull * VEC)) - 1u) & ((1u << VEC) - 1u)) : 0u;
  const int nw = (nval + 31) >> 5;                                // bitmap words of the chunk
  const uint8_t* lg = reinterpret_cast<const uint8_t*>(a.logits);

  if (tid == 0) {
    for (int b = 0; b < kRNB; ++b) {
      mbar_init(full + b, 1);
      mbar_init(empty + b, kSW);
    }
    for (int s2 = 0; s2 < kNS; ++s2) {
      mbar_init(spass + s2, kSW);
      mbar_init(sfree + s2, 1);
    }
    for (int f = 0; f < kNF; ++f) mbar_init(bound + f, C);
    mbar_init(recfull, C);
    for (int l = 0; l < kRCMax; ++l) mbar_init(slotfree + l, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < kNS; i += blockDim.x) {  // summary slots start empty
    SlotHdr* sh = reinterpret_cast<SlotHdr*>(smem + L.sl + i * L.slb);
    sh->npen = 0;
    sh->bad = 0;
  }
  // the previous kernel of the stream (the last step, which appended to the histories) is complete
  // before any memory access; the next step may be scheduled as this grid retires
  griddep_wait();
  griddep_launch();
  cl_sync();  // every CTA's barriers are initialised before any remote arrive

  if (warp == kRProdW) {
    // ================= producer: bulk copies of this CTA's chunk of each row =================
    if (lane == 0 && nrows > 0) {
      // L2 evict-normal: the finishers re-read the few candidate groups of a chunk from L2
      const uint32_t dbytes = (uint32_t)((nval * ESZ + 15) / 16 * 16);
      const uint32_t bmb = (uint32_t)((nval + 127) / 128 * 16);
      for (int it = 0; it < nrows; ++it) {
        const int b = it % kRNB;
        if (it >= kRNB) mbar_wait_sleep(empty + b, (uint32_t)((it / kRNB - 1) & 1));
        RTR(it, 0);
        const int64_t r = (int64_t)q + (int64_t)it * nclus;
        RowStage* st = reinterpret_cast<RowStage*>(smem + L.stg) + b;
        if (nval > 0) {  // the logits first: they do not depend on the slot
          mbar_expect_tx(full + b, dbytes + bmb);
          bulk_g2s_nohint(smem + L.buf + b * a.Lc * ESZ, lg + (r * a.ld + c0) * ESZ, dbytes, full + b);
        }
        const int slot = a.slots ? a.slots[r] : (int)r;
        if (nval > 0)
          bulk_g2s_nohint(smem + L.bm + b * (a.Lc / 8), a.hs.pmask + (int64_t)slot * a.hs.pmw + c0 / 32, bmb,
                          full + b);
        st->prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
        st->slot = slot;
        mbar_arrive(full + b);  // (release: the staged row info above)
        RTR(it, 1);
      }
    }
  } else if (warp == kRDecW) {
    // ================= decider: the rows this CTA leads (row index it with it % C == rank) =========
    MergeSmem ms;
    ms.pool = reinterpret_cast<uint64_t*>(smem + L.pool);
    ms.top = reinterpret_cast<uint64_t*>(smem + L.top);
    ms.wv = reinterpret_cast<double*>(smem + L.wv);
    ms.byid = reinterpret_cast<uint64_t*>(smem + L.byid);
    ms.hdr = nullptr;
    ms.off = nullptr;
    uint8_t* dsc = smem + L.dscr;
    ms.bs.f = reinterpret_cast<float*>(dsc);
    ms.bs.d = reinterpret_cast<double*>(dsc + 32);
    ms.bs.u = reinterpret_cast<uint64_t*>(dsc + 96);
    ms.bs.i = reinterpret_cast<int*>(dsc + 224);
    const RecC* hdr = reinterpret_cast<const RecC*>(smem + L.hdr);
    const uint64_t* rec = reinterpret_cast<const uint64_t*>(smem + L.rec);
    const RowStage* ri = reinterpret_cast<const RowStage*>(smem + L.rinfo);
    for (int it = (int)rank; it < nrows; it += C) {
      const int r = (int)q + it * (int)nclus;
      mbar_wait_cl(recfull, (uint32_t)((it / C) & 1));
      if (lane == 0) RTR(it, 12);
      const sampling_params prm = ri->prm;
      const int slot = ri->slot;
      const RowCfg rc = decode_row(prm, a.V, a.kcand);
      const bool bounded = rc.greedy || (rc.topk_on && rc.k <= a.kcand);
      const int keff = rc.keff;
      // M, S, frontier, flags: lane c holds chunk c (fixed order: deterministic)
      const bool has = lane < C;
      RecC h;
      if (has) h = hdr[lane];
      const float M = warp_max(has ? h.m : -INFINITY);
      const double term = (has && h.s != 0.0) ? h.s * exp2(((double)h.m - (double)M) * rc.c_d) : 0.0;
      const double S = warp_sum_d(term);
      uint64_t F = warp_max_u64(has ? h.front : 0ull);
      const bool bad = __any_sync(kFull, has && (h.flags & 1u));
      const bool ovf = __any_sync(kFull, has && (h.flags & 2u));  // a chunk list overflowed (massive ties)
      const uint64_t best = warp_max_u64(has ? h.best : 0ull);
      // the candidates of the C chunks (every element of the row >= the row bound, unsorted) into the
      // pool, then the exact top-keff by rank counting (composites are unique)
      const int nc = has ? h.n : 0;
      const int ninc = warp_incl_scan_i(nc, lane);
      const int tot = __shfl_sync(kFull, ninc, 31);  // (<= C * cap)
      int n = 0;
      if (!rc.greedy) {
        for (int c = 0, base = 0; c < C; ++c) {
          const int ncc = hdr[c].n;
          for (int i = lane; i < ncc && base + i < tot; i += 32) ms.pool[base + i] = rec[c * a.cap + i];
          base += ncc;
        }
        __syncwarp();
        n = warp_topk(ms.pool, tot, keff, reinterpret_cast<uint64_t*>(ms.wv), ms.top, lane);
      }
      __syncwarp();
      // the chunk lists are consumed: release every sender's slot for this leader
      if (lane < C) cl_arrive_remote(cl_map(smem_u32(slotfree + rank), (uint32_t)lane));
      if (rc.greedy) {
        if (lane == 0) ms.top[0] = best;
        __syncwarp();
        n = (best != 0ull) ? 1 : 0;
        F = best;
      } else if (tot > keff && n > 0) {
        const uint64_t last = ms.top[n - 1];
        F = last > F ? last : F;
      }
      if (lane == 0) RTR(it, 13);
      const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
      if (a.mode == 1) {  // vocab-sharded phase 1: the row's candidate record (merge.cuh)
        uint8_t* out = a.out_records + (int64_t)r * a.out_stride;
        uint64_t* oe = reinterpret_cast<uint64_t*>(out + kRecHdrBytes);
        for (int i = lane; i < n; i += 32) oe[i] = ms.top[i];
        if (lane == 0) {
          RecHdr o;
          o.m = M;
          o.flags = bad ? kRecBad : 0u;
          o.s = S;
          o.R = (double)M * rc.c_d;
          o.n = (uint32_t)n;
          o.rsv = 0;
          o.frontier = ovf ? ~0ull : F;
          *reinterpret_cast<RecHdr*>(out) = o;
        }
        __syncwarp();
        continue;
      }
      if (!bounded || ovf) {  // exact.cuh finishes the row from {M, S}
        if (lane == 0) {
          RowInfo o;
          o.M = M;
          o.status = bad ? SAMPLER_ROW_NONFINITE : (M > -INFINITY ? kRowPending : SAMPLER_ROW_ALL_NEG_INF);
          o.S = S;
          o.W = 0.0;
          o.cutoff = 0;
          o.token = -1;
          o.greedy = rc.greedy;
          a.ro.info[r] = o;
          if (o.status != kRowPending) {
            a.ro.tokens[r] = -1;
            a.ro.logprobs[r] = NAN;
            if (a.ro.flogprobs) a.ro.flogprobs[r] = NAN;
            if (a.ro.status) a.ro.status[r] = o.status;
          }
        }
        __syncwarp();
        continue;
      }
      const int tok = warp_decide(ms, n, M, S, F, bad, rc, prm, seed, a.step, r, a.ro, false, nullptr);
      if (a.append && tok >= 0 && lane == 0) hist_append(a.hs, slot, tok);
      if (lane == 0) RTR(it, 14);
      __syncwarp();
    }
  } else if (warp < kSW) {
    // ================= stream warps: the pass over each chunk (no block barrier) =================
    const int t = tid;
    const uint4 kNegVec = make_uint4(VEC == 8 ? 0xFF80FF80u : 0xFF800000u, VEC == 8 ? 0xFF80FF80u : 0xFF800000u,
                                     VEC == 8 ? 0xFF80FF80u : 0xFF800000u, VEC == 8 ? 0xFF80FF80u : 0xFF800000u);
    uint32_t* pme = reinterpret_cast<uint32_t*>(smem + L.pme) + t * kPT;  // this thread's staged counts
    const int wpt = (nw + kST - 1) / kST;                                  // bitmap words per thread
    const int w0 = min(nw, t * wpt), w1 = min(nw, w0 + wpt);
    for (int it = 0; it < nrows; ++it) {
      const int b = it % kRNB, sidx = it % kNS;
      const uint8_t* buf = smem + L.buf + b * a.Lc * ESZ;
      const uint4* buf4 = reinterpret_cast<const uint4*>(buf);
      const uint8_t* bm = smem + L.bm + b * (a.Lc / 8);
      const uint32_t* bmw = reinterpret_cast<const uint32_t*>(bm);
      uint8_t* sl = smem + L.sl + sidx * L.slb;
      SlotHdr* sh = reinterpret_cast<SlotHdr*>(sl);
      float* s_tmax = reinterpret_cast<float*>(sl + sizeof(SlotHdr));
      float* s_mref = s_tmax + kST;
      float* s_ssum = s_mref + kST;
      uint8_t* s_keys = reinterpret_cast<uint8_t*>(s_ssum + kST);
      int2* s_pen = reinterpret_cast<int2*>(s_keys + ((a.Lc / 16) * (ESZ == 2 ? 2 : 4) + 15) / 16 * 16);
      // the summary slot must be released by the finisher of the row kNS before
      if (it >= kNS) mbar_wait_sleep(sfree + sidx, (uint32_t)((it / kNS - 1) & 1));
      mbar_wait_sleep(full + b, (uint32_t)((it / kRNB) & 1));
      if (t == 0) RTR(it, 2);
      const RowStage* st = reinterpret_cast<const RowStage*>(smem + L.stg) + b;
      const sampling_params prm = st->prm;
      const int slot = st->slot;
      if (t == 0) {
        sh->prm = prm;
        sh->slot = slot;
      }
      const float temp = prm.temperature;
      const float tau = (temp < kGreedyEps) ? 1.0f : temp;
      const float cf = __fdiv_rn((float)kLog2e, tau);
      const float inv8 = __fdiv_rn(8.0f, cf);
      const uint32_t* gme = a.hs.pmeta + (int64_t)slot * a.hs.vls + c0;
      // penalised ids of this thread's bitmap words: counts gathered behind the pass (LDGSTS)
      int pl[kPT];
      int npt = 0;
      for (int w = w0; w < w1; ++w) {
        uint32_t bits = bmw[w];
        while (bits) {
          const int l = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          if (npt < kPT) {
#pragma unroll
            for (int j = 0; j < kPT; ++j)
              if (j == npt) pl[j] = l;
            cp_async4(pme + npt, gme + l);
          }
          ++npt;
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // ---- the pass: 2 vectors (a "group", <= 16 elements) per iteration.  Per group its max
      //      (NaN-propagating; its key kept for the finisher's candidate re-read); the exp-sum of
      //      P:149's softmax denominator relative to the thread's reference m_ref, rebased only
      //      when a group max exceeds it by 8/c (every term <= 2^8).  Penalised ids and the
      //      ragged tail are masked to -inf (the penalised ones enter below as exact values).
      float tmax = -INFINITY, mref = -INFINITY, thr = -INFINITY;
      float ssum = 0.f;
      uint32_t bad = 0;
      {
        uint64_t c2;
        asm("mov.b64 %0, {%1, %2};" : "=l"(c2) : "f"(cf), "f"(cf));
        for (int v = t, k = t; v < nvec; v += 2 * kST, k += kST) {
          uint4 u0 = buf4[v];
          uint4 u1 = (v + kST < nvec) ? buf4[v + kST] : kNegVec;
          const uint32_t b0 = vec_bits<VEC>(bm, v) | (v == nfull ? tailmask : 0u);
          const uint32_t b1 = (v + kST < nvec) ? (vec_bits<VEC>(bm, v + kST) | (v + kST == nfull ? tailmask : 0u)) : 0u;
          if (b0) u0 = RV<T>::mask(u0, b0);
          if (b1) u1 = RV<T>::mask(u1, b1);
          float gm;
          if (VEC == 8) {
            const __nv_bfloat162 m2 =
                __hmax2_nan(RV<__nv_bfloat16>::vmax2_nan(u0), RV<__nv_bfloat16>::vmax2_nan(u1));
            gm = fmax_nan(__low2float(m2), __high2float(m2));
            reinterpret_cast<uint16_t*>(s_keys)[k] = (uint16_t)(__float_as_uint(gm) >> 16);
          } else {
            gm = fmax_nan(RV<float>::vmax_nan(u0), RV<float>::vmax_nan(u1));
            reinterpret_cast<uint32_t*>(s_keys)[k] = __float_as_uint(gm);
          }
          tmax = fmax_nan(tmax, gm);
          if (gm > thr) {  // (rare) rebase; also the thread's first finite group
            if (ssum != 0.f) ssum *= ex2f(__fmul_rn(mref - gm, cf));
            mref = gm;
            thr = gm + inv8;
          }
          if (mref > -INFINITY) ssum += RV<T>::esum(u0, -mref, cf, c2) + RV<T>::esum(u1, -mref, cf, c2);
        }
      }
      if (t == 0) RTR(it, 3);
      // ---- this thread's penalised values (exact binary32 penalty, P:146 / P:371): into the max,
      //      the sum and the slot's penalised list
      cp_async_wait_all();
      auto pen = [&](int l, float zp) {
        if (!(zp < INFINITY)) {  // NaN / +inf
          bad = 1;
          return;
        }
        if (zp > -INFINITY) {
          tmax = fmaxf(tmax, zp);
          if (zp > thr) {
            if (ssum != 0.f) ssum *= ex2f(__fmul_rn(mref - zp, cf));
            mref = zp;
            thr = zp + inv8;
          }
          ssum += ex2f(__fmul_rn(__fsub_rn(zp, mref), cf));
        }
        const int e = atomicAdd(&sh->npen, 1);
        if (e < kPenS) s_pen[e] = make_int2(a.voff + c0 + l, __float_as_int(zp));
      };
#pragma unroll
      for (int j = 0; j < kPT; ++j)
        if (j < npt) pen(pl[j], apply_penalty(RV<T>::at(buf, pl[j]), pme[j], prm, a.pen_mode));
      if (npt > kPT) {
        int j = 0;
        for (int w = w0; w < w1; ++w) {
          uint32_t bits = bmw[w];
          while (bits) {
            const int l = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            if (j++ >= kPT) pen(l, apply_penalty(RV<T>::at(buf, l), gme[l], prm, a.pen_mode));
          }
        }
      }
      if (tmax != tmax || tmax == INFINITY) bad = 1;
      if (__any_sync(kFull, bad) && lane == 0) atomicOr(&sh->bad, 1);
      s_tmax[t] = tmax;
      s_mref[t] = mref;
      s_ssum[t] = ssum;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty + b);    // the chunk buffer is free for the producer
        mbar_arrive(spass + sidx); // (release: this warp's summary entries)
      }
    }
  } else {
    // ================= finisher groups: rows it = f, f + kNF, ... ==========================
    const int f = (warp - kSW) / kFW;
    const int ft = tid - (kSW + f * kFW) * 32, fw = ft >> 5;
    uint8_t* fsc = smem + L.fscr + f * kFScrBytes;
    uint64_t* lc = reinterpret_cast<uint64_t*>(fsc);           // [kRCapL] candidates
    uint8_t* fs = fsc + kRCapL * 8;
    uint32_t* f_m = reinterpret_cast<uint32_t*>(fs);           // [4] max keys
    uint32_t* f_t = reinterpret_cast<uint32_t*>(fs + 16);      // [1] the chunk bound
    double* f_s = reinterpret_cast<double*>(fs + 32);          // [4] sums
    uint64_t* f_b = reinterpret_cast<uint64_t*>(fs + 64);      // [4] greedy best
    int* f_cnt = reinterpret_cast<int*>(fs + 96);              // [1] candidate count
    const int pmw = a.hs.pmw;
    for (int it = f; it < nrows; it += kNF) {
      const int sidx = it % kNS, par = (it / kNF) & 1;
      const int r = (int)q + it * (int)nclus;
      const int leader = it % C;
      uint8_t* sl = smem + L.sl + sidx * L.slb;
      SlotHdr* sh = reinterpret_cast<SlotHdr*>(sl);
      const float* s_tmax = reinterpret_cast<const float*>(sl + sizeof(SlotHdr));
      const float* s_mref = s_tmax + kST;
      const float* s_ssum = s_mref + kST;
      const uint8_t* s_keys = reinterpret_cast<const uint8_t*>(s_ssum + kST);
      const int2* s_pen = reinterpret_cast<const int2*>(s_keys + ((a.Lc / 16) * (ESZ == 2 ? 2 : 4) + 15) / 16 * 16);
      mbar_wait_sleep(spass + sidx, (uint32_t)((it / kNS) & 1));
      if (ft == 0) RTR(it, 4);
      const sampling_params prm = sh->prm;
      const int slot = sh->slot;
      const RowCfg rc = decode_row(prm, a.V, a.kcand);
      const int keff = rc.keff;
      const float cf = __fdiv_rn((float)kLog2e, rc.tau);
      const bool badc = sh->bad != 0;
      // ---- chunk max (the stream threads' maxima include the penalised values)
      float tm[kST / kFT];
      float mloc = -INFINITY;
#pragma unroll
      for (int j = 0; j < kST / kFT; ++j) {
        tm[j] = s_tmax[ft + j * kFT];
        mloc = fmaxf(mloc, tm[j]);
      }
      const uint32_t mk = __reduce_max_sync(kFull, f2key(mloc));
      if (lane == 0) f_m[fw] = mk;
      if (ft == 0) *f_cnt = 0;
      fbar(f);
      uint32_t mkey = f_m[0];
#pragma unroll
      for (int j = 1; j < kFW; ++j) mkey = max(mkey, f_m[j]);
      const float mc = key2f(mkey);  // chunk max (-inf if empty)
      const bool live = !badc && mc > -INFINITY;
      // ---- S_c relative to the chunk max (fixed order: deterministic)
      double ss = 0.0;
      if (live) {
#pragma unroll
        for (int j = 0; j < kST / kFT; ++j) {
          const int tt = ft + j * kFT;
          const float sv = s_ssum[tt];
          if (sv != 0.f) ss += (double)sv * (double)ex2f(__fmul_rn(s_mref[tt] - mc, cf));
        }
      }
      ss = warp_sum_d(ss);
      if (lane == 0) f_s[fw] = ss;
      // ---- the chunk bound T_c = the keff-th largest stream-thread max (keff distinct elements are
      //      >= T_c; a lower bound of the row's keff-th largest z'): warp 0, bitwise radix select
      if (fw == 0) {
        uint32_t k[kST / 32];
#pragma unroll
        for (int j = 0; j < kST / 32; ++j) {
          const float x = s_tmax[lane + 32 * j];
          k[j] = (live && x > -INFINITY && x < INFINITY) ? f2key(x) : 0u;
        }
        uint32_t pre = 0;
#pragma unroll 1
        for (int bb = 31; bb >= 0; --bb) {
          const uint32_t cand = pre | (1u << bb);
          uint32_t c = 0;
#pragma unroll
          for (int j = 0; j < kST / 32; ++j) c += (k[j] >= cand) ? 1u : 0u;
          if ((int)__reduce_add_sync(kFull, c) >= keff) pre = cand;
        }
        if (lane == 0) *f_t = pre;
      }
      fbar(f);
      const uint32_t tkey = *f_t;
      // ---- the row bound: every CTA's chunk bound to every CTA of the cluster (DSMEM), T = the max
      //      (each is a lower bound of the row's keff-th largest, so the max is too); candidates are
      //      then only the row's elements >= T, about keff of them in the cluster
      uint32_t* bs = reinterpret_cast<uint32_t*>(smem + L.bslot) + (f * 2 + par) * kRCMax;
      if (ft < C) {
        const uint32_t dst = cl_map(smem_u32(bs + rank), (uint32_t)ft);
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(dst), "r"(tkey) : "memory");
        cl_arrive_remote(cl_map(smem_u32(bound + f), (uint32_t)ft));
      }
      mbar_wait_cl(bound + f, (uint32_t)par);
      if (ft == 0) RTR(it, 5);
      uint32_t rkey = 0;
      for (int c = 0; c < C; ++c) rkey = max(rkey, bs[c]);
      const float Tf = rkey ? key2f(rkey) : -INFINITY;
      // ---- candidates: the stream threads whose max reaches T, their groups whose key reaches T
      //      re-read from L2 (the chunk buffer is already refilled), every element >= T listed
      uint64_t tbest = 0ull;
      auto push = [&](float z, int gid) {
        const uint64_t cmp = make_comp(z, gid);
        if (rc.greedy) {
          tbest = cmp > tbest ? cmp : tbest;
        } else {
          const int at = atomicAdd(f_cnt, 1);
          if (at < kRCapL) lc[at] = cmp;
        }
      };
      if (live) {
        const uint8_t* grow = lg + ((int64_t)r * a.ld + c0) * ESZ;
        const uint32_t* gpm = a.hs.pmask + (int64_t)slot * pmw + c0 / 32;
#pragma unroll
        for (int j = 0; j < kST / kFT; ++j) {
          if (!(tm[j] >= Tf)) continue;
          const int tt = ft + j * kFT;
          for (int v = tt, k = tt; v < nvec; v += 2 * kST, k += kST) {
            const float gm = (ESZ == 2) ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(s_keys)[k] << 16)
                                        : __uint_as_float(reinterpret_cast<const uint32_t*>(s_keys)[k]);
            if (!(gm >= Tf && gm > -INFINITY)) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int vv = v + h * kST;
              if (vv >= nvec) continue;
              uint4 u = *reinterpret_cast<const uint4*>(grow + (int64_t)vv * 16);
              const int e0 = vv * VEC;
              uint32_t pb = (gpm[e0 >> 5] >> (e0 & 31)) & ((1u << VEC) - 1u);
              if (vv == nfull) pb |= tailmask;
              if (pb) u = RV<T>::mask(u, pb);
#pragma unroll
              for (int q2 = 0; q2 < VEC; ++q2) {
                const float z = RV<T>::elem(u, q2);
                if (z >= Tf && z > -INFINITY) push(z, a.voff + c0 + e0 + q2);
              }
            }
          }
        }
        const int npen = sh->npen;
        if (npen <= kPenS) {
          for (int e = ft; e < npen; e += kFT) {
            const int2 pe = s_pen[e];
            const float zp = __int_as_float(pe.y);
            if (zp >= Tf && zp > -INFINITY) push(zp, pe.x);
          }
        } else {  // long histories: every penalised id of the chunk again, from global memory
          const uint32_t* gme = a.hs.pmeta + (int64_t)slot * a.hs.vls + c0;
          for (int w = ft; w < nw; w += kFT) {
            uint32_t bits = gpm[w];
            while (bits) {
              const int l = w * 32 + __ffs(bits) - 1;
              bits &= bits - 1;
              const float x = (ESZ == 2) ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(grow)[l] << 16)
                                         : reinterpret_cast<const float*>(grow)[l];
              const float zp = apply_penalty(x, gme[l], prm, a.pen_mode);
              if (zp >= Tf && zp > -INFINITY && zp < INFINITY) push(zp, a.voff + c0 + l);
            }
          }
        }
      }
      tbest = warp_max_u64(tbest);
      if (lane == 0) f_b[fw] = tbest;
      // the leader's list for this row must be free before this chunk's list is written into it
      if (ft == 0 && it >= C) mbar_wait_cl(slotfree + leader, (uint32_t)((it / C - 1) & 1));
      fbar(f);
      // the summary slot is consumed
      if (ft == 0) {
        sh->npen = 0;
        sh->bad = 0;
        mbar_arrive(sfree + sidx);
      }
      const int cnt = *f_cnt;
      const bool over = !rc.greedy && cnt > a.cap;  // (massive ties: exact.cuh finishes the row)
      const int nout = (rc.greedy || over) ? 0 : cnt;
      const uint32_t rec_remote = cl_map(smem_u32(smem + L.rec), (uint32_t)leader) + rank * (uint32_t)(a.cap * 8);
      for (int i = ft; i < nout; i += kFT) cl_st64(rec_remote + (uint32_t)i * 8u, lc[i]);
      fbar(f);
      if (ft == 0) {
        RecC h;
        h.m = mc;
        h.flags = (badc ? 1u : 0u) | (over ? 2u : 0u);
        double s2 = 0.0;
        uint64_t bb = 0ull;
#pragma unroll
        for (int j = 0; j < kFW; ++j) {
          s2 += f_s[j];
          bb = f_b[j] > bb ? f_b[j] : bb;
        }
        h.s = s2;
        h.front = rkey ? make_comp(Tf, 0x7FFFFFFF) : 0ull;
        h.best = bb;
        h.n = nout;
        h.pad[0] = h.pad[1] = h.pad[2] = 0;
        const uint32_t hr = cl_map(smem_u32(smem + L.hdr), (uint32_t)leader) + rank * (uint32_t)sizeof(RecC);
        const uint4* hv = reinterpret_cast<const uint4*>(&h);
#pragma unroll
        for (int j = 0; j < (int)(sizeof(RecC) / 16); ++j) cl_st128(hr + 16 * j, hv[j]);
        if (rank == (uint32_t)leader) {  // the row's params / slot for the decider
          RowStage* rs = reinterpret_cast<RowStage*>(smem + L.rinfo);
          rs->prm = prm;
          rs->slot = slot;
        }
        cl_fence();  // the group's list entries (ordered before this thread by the barrier) and the header
        cl_arrive_remote(cl_map(smem_u32(recfull), (uint32_t)leader));
        RTR(it, 7);
        RTV(it, 8, cnt);
        RTV(it, 9, tkey);
        RTV(it, 10, rkey);
      }
    }
  }
  __syncwarp();
  cl_sync();  // no CTA leaves while another may still address its shared memory
}

}  // namespace smp

// common.cuh — device helpers for the sm_100a sampler kernels.
//
// Nothing here is shared with oracle/ (the CPU checker); the two are independent
// statements of the same definition.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/sampler.h"

#ifndef SAMPLER_KCAND_MAX
#define SAMPLER_KCAND_MAX 128
#endif

namespace smp {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr float kGreedyEps = 1e-5f;       // DESIGN.md R5: tau < 1e-5 => greedy
constexpr double kLog2e = 1.4426950408889634073599246810019;
constexpr double kLn2 = 0.69314718055994530941723212145818;

// ---- per-slot state (device) --------------------------------------------------------
struct SlotMeta {
  int32_t n_prompt;
  int32_t n_out;
  int32_t n_uniq;
  int32_t flags;  // bit0: history overflow happened (append dropped)
};

// Unique-token penalty entry: id ascending; meta = (count_in_output << 1) | in_prompt.
// This is the device form of the paper's incremental penalty buffer f: only the
// entries of tokens that occurred are stored (sparse), updated in place on append.
struct __align__(8) UniqEntry {
  int32_t id;
  uint32_t meta;
};

// ---- partial-reduction record (piece / rank) ----------------------------------------
// A record summarises one contiguous vocabulary range of one row:
//   m   = max z' over the range (binary32), s = sum 2^((z'-m)*c) (float64),
//   list = the range's top-K candidates as composites (see below), exact down to `frontier`:
//          every element of the range with composite >= frontier is in the list.
struct __align__(16) RecHdr {
  float m;          // max z' over the range (binary32)
  uint32_t flags;   // bit0 bad (NaN/+inf seen)
  double s;         // sum over the range of 2^(z'*log2(e)/tau - R)
  double R;         // exponent reference of s
  uint32_t n;       // entries in the list (sorted descending)
  uint32_t rsv;
  uint64_t frontier;  // every element with composite >= frontier is in the list (0: all)
};
static_assert(sizeof(RecHdr) == 48, "RecHdr layout");
constexpr int kRecHdrBytes = 48;

constexpr uint32_t kRecBad = 1u;

__host__ __device__ inline int64_t rec_stride_bytes(int kcand) {
  return (int64_t)kRecHdrBytes + 8 * (int64_t)kcand;
}
__device__ __forceinline__ const uint64_t* rec_entries(const uint8_t* rec) {
  return reinterpret_cast<const uint64_t*>(rec + kRecHdrBytes);
}

// Per-row result / hand-off info (unresolved rows, debug distribution).
struct __align__(16) RowInfo {
  float M;          // row max of z'
  int32_t status;   // SAMPLER_ROW_* ; kRowPending = needs the exact multi-pass kernel
  double S;         // sum exp((z'-M)/tau_eff)
  double W;         // mass of the kept set K3
  uint64_t cutoff;  // K3 = { composite >= cutoff }
  int32_t token;
  int32_t greedy;
};
constexpr int32_t kRowPending = 100;

// ---- NEXT-2: one-shot peer exchange of the vocab-sharded records (sampler_sample_exchange) ----
// Every rank owns one exchange buffer: [2 parities][world ranks][B_max rows][rec_stride] records
// followed by [world][B_max] u32 flags.  Rank q's phase 1 stores row r's record straight into every
// peer's buffer (NVLink P2P stores through IPC-mapped pointers) at (parity, q, r) and then raises
// flag (q, r) of every peer to the row's sequence number (release, system scope); a peer's merge
// waits for flag (q, r) >= its own sequence number for every q (acquire) and reads its local copy.
// seq[r] counts the exchanges of batch row r on this handle (all ranks make the same calls, so
// the numbers agree); parity = seq & 1 double-buffers the records (a rank runs at most one step
// ahead of a peer: its next merge waits for that peer's next phase 1).
struct ExchPeers {
  uint8_t* const* bases;  // [world] device pointers (this process' mappings of every rank's buffer)
  int world, rank;
  int64_t row_stride;     // rec_stride
  int64_t rank_pitch;     // B_max * rec_stride
  int64_t par_pitch;      // world * rank_pitch
  int64_t flags_off;      // bytes from a base to its flags
  int nslots;             // B_max
  uint32_t* seq;          // [B_max] local sequence numbers of phase 1 (publish)
  uint32_t* mseq;         // [B_max] local sequence numbers of the merge (the same count)
  uint64_t timeout_ns;
  int64_t region_off;     // bytes from a base to this region (records: 0; resolve payloads: after them)
};
// flag store / load: system scope across GPUs (NVLink peers), GPU scope when every rank is this GPU
__device__ __forceinline__ void st_release_flag(uint32_t* p, uint32_t v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_flag(const uint32_t* p, bool sys) {
  uint32_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- order-preserving keys ----------------------------------------------------------
// key(f) is monotone in f (as a float, -0 canonicalised to +0 so that equal values tie);
// composite = key << 32 | (0xFFFFFFFF - id) orders by (z' desc, id asc) when sorted
// descending — the order pi of DESIGN.md R9.
__device__ __forceinline__ uint32_t f2key(float f) {
  f = f + 0.0f;  // -0 -> +0 (IEEE: -0 + +0 = +0 in round-to-nearest)
  uint32_t u = __float_as_uint(f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = k ^ ((k >> 31) ? 0x80000000u : 0xFFFFFFFFu);
  return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t make_comp(float z, int32_t id) {
  return ((uint64_t)f2key(z) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)id);
}
__device__ __forceinline__ int32_t comp_id(uint64_t c) {
  return (int32_t)(0xFFFFFFFFu - (uint32_t)(c & 0xFFFFFFFFu));
}
__device__ __forceinline__ float comp_val(uint64_t c) { return key2f((uint32_t)(c >> 32)); }

// ---- PTX wrappers: mbarrier + 1-D bulk async copy (TMA engine) ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// wait with back-off: a warp whose tile is not ready sleeps between polls instead of spinning on
// the issue port (the consumer warps of a CTA share their sub-partitions with the busy ones)
#ifndef SMP_SLEEP_NS
#define SMP_SLEEP_NS 128  // back-off of the ring waits (tools/variants.py: 32-512 tried)
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns = SMP_SLEEP_NS) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}
#ifndef SMP_L2POL
#define SMP_L2POL 0
#endif
// L2 policy of phase A's logits copies: 0 evict_first (default), 1 evict_normal, 2 evict_last
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
#if SMP_L2POL == 1
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#elif SMP_L2POL == 2
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
// global -> shared bulk copy without an L2 cache hint
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// exp2 on the MUFU (ex2.approx.ftz.f32): |rel err| ~ 2^-22
// programmatic dependent launch: the dependent grid may start; wait for the primary grid
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// named barrier 2 among the first N threads of the CTA (warp-specialised kernels)
template <int N>
__device__ __forceinline__ void cbar_n() {
  asm volatile("bar.sync 2, %0;" ::"n"(N) : "memory");
}

// ---- warp collectives ---------------------------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    uint64_t t = __shfl_xor_sync(kFull, v, o);
    v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    uint64_t t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  return v;
}
// inclusive prefix sum over lanes
__device__ __forceinline__ int warp_incl_scan_i(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ double warp_incl_scan_d(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// ---- per-row parameter decode ------------------------------------------------------
struct RowCfg {
  int greedy;
  int topk_on;   // 1 <= k < V
  int k;
  float tau;     // tau_eff (1 for greedy)
  float top_p;
  float min_p;
  int keff;      // candidates tracked per partial reduction
  double c_d;    // log2(e) / tau_eff
  float c_hi, c_lo;
  float delta;   // rescale margin in logit units: 8 / c  (w <= 2^8 before a rescale)
};

__device__ __forceinline__ RowCfg decode_row(const sampling_params& p, int V, int kcand) {
  RowCfg r;
  r.greedy = p.temperature < kGreedyEps;
  r.tau = r.greedy ? 1.0f : p.temperature;
  r.topk_on = (p.top_k >= 1 && p.top_k < V);
  r.k = p.top_k;
  r.top_p = p.top_p;
  r.min_p = p.min_p;
  if (r.greedy)
    r.keff = 1;
  else if (r.topk_on)
    r.keff = p.top_k < kcand ? p.top_k : kcand;
  else
    r.keff = kcand;
  r.c_d = kLog2e / (double)r.tau;
  // two-term log2(e)/tau with c_lo > 0 (c_hi rounded down) so that -inf * c_lo never makes
  // +inf and (-inf)*c_hi + (-inf)*c_lo stays -inf for -inf logits / sentinels
  r.c_hi = __double2float_rd(r.c_d);
  r.c_lo = fmaxf((float)(r.c_d - (double)r.c_hi), 1e-30f);
  r.delta = (float)(8.0 / r.c_d);
  return r;
}

}  // namespace smp

// stream.cuh — phase A of the sampling step: one streaming pass over the logits [B x V].
//
// Persistent CTAs (one per SM), warp-specialised.  The padded step space [B x Vq/128] (a step =
// 128 16-byte vectors = 2 KB of one row) is cut into equal contiguous CTA spans:
//   * producer warp: one 1-D bulk copy (cp.async.bulk, TMA engine, L2 evict-first) per step into a
//     ring of kNS tiles of 16 steps (32 KB each), full / empty mbarriers;
//     next to each run of logits, the same steps' words of the slot's penalty presence bitmap
//     (HistState::pmask — the support of the paper's incremental penalty buffers);
//   * 26 consumer warps: warp w takes step w of every tile (4 vectors = 32 bf16 / 16 f32 logits per
//     lane); penalised ids and the padding tail are masked to -inf in registers (the penalised
//     elements enter phase B as exact single values); then per lane and step (a "group"):
//       - the group max by a NaN-propagating packed max tree (bf16x2 HMNMX2), its order-preserving
//         16-bit key stored to gkeys[row][group] (phase B selects the top-k from these keys);
//       - the exp-sum of P:149's softmax denominator, sum 2^((z - m_ref) * log2(e)/tau):
//         bf16: t = z - m_ref straight from the packed register half (mixed-precision FHFMA.BF16,
//         exact for bf16 operands), x = t * c by packed FMUL2, MUFU.EX2, packed FADD2 tree, one
//         float64 add per group.  m_ref (lane-private) is rebased only when a group max exceeds
//         it by 8 / c (every term <= 2^8), the float64 sum rescaled by exp2 in float64.
//   * when a warp leaves a row: its partial record {max m, s = sum 2^((z - m) log2(e)/tau)
//     (float64), bad} (phase B adds the penalised elements as exact single values).
// The selection (bound from the group keys, re-read of the qualifying groups, exact top-K,
// decision, draw) is phase B (select.cuh).
#pragma once
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "piece.cuh"

namespace smp {

// ---- geometry of phase A (persistent CTAs, warp-specialised) ----------------------
#ifndef SMP_KCW
#define SMP_KCW 26
#endif
#ifndef SMP_KNS
#define SMP_KNS 3
#endif
constexpr int kCW = SMP_KCW;               // consumer warps per CTA (one step of each tile each)
constexpr int kStreamCtasPerSm = 1;        // CTAs (independent pipelines) per SM
constexpr int kTileSteps = kCW;            // steps per ring tile (26 x 2 KB = 52 KB)
constexpr int kNS = SMP_KNS;               // ring tiles (3 x 52 KB; 3 beat 4 and 2 at c3: tools/variants.py)
constexpr int kMaxSeg = 48;                // rows per CTA span (the host caps the span)
constexpr int kStreamThreads = (kCW + 2) * 32;  // + producer warp + penalty warp
constexpr int kStepBytes = kStepVec * 16;
constexpr int kSOffRing = 0;
constexpr int kSOffBm = kSOffRing + kNS * kTileSteps * kStepBytes;  // [kNS][kTileSteps][32] u32
constexpr int kSOffBar = kSOffBm + kNS * kTileSteps * 128;
constexpr int kSOffSeg = kSOffBar + 2 * kNS * 8;
constexpr int kPenB = 1024;                 // penalty hand-off: table entries per batch (32 per lane)
constexpr int kSOffPen = kSOffSeg + kMaxSeg * 8;                     // [2][kPenB + 2] UniqEntry (TMA-staged)
constexpr int kSOffPenBar = kSOffPen + 2 * (kPenB + 2) * 8;          // 2 mbarriers
constexpr int kStreamSmem = kSOffPenBar + 2 * 8;

// Phase A -> phase B hand-off of one batch row, written by the CTA that holds the row's first step
// (its penalty warp), so that phase B starts with one round trip and no slot indirection:
// the slot, its history meta, the row's params and, per unique history entry (id order), the
// exact penalised logit z' (R1-R3).
struct __align__(16) RowHand {
  int32_t slot;
  int32_t pad[3];
  SlotMeta meta;
  sampling_params prm;
};
struct __align__(16) PenEnt {
  int32_t id;
  uint32_t meta;  // (count in output << 1) | in prompt
  float zp;       // penalised logit (only for ids inside the local slice)
  int32_t pad;
};

// one consumer warp's partial reduction of one row: max m and s = sum 2^((z - m) log2(e)/tau)
struct __align__(16) PartRec {
  float m;
  uint32_t bad;
  double s;
};

struct StreamArgs {
  const void* logits;
  int64_t ld;          // row stride (elements)
  int B;
  int V;               // global vocab
  int voff, vloc;      // local slice
  int64_t Vq;          // padded row length in vectors (multiple of kStepVec)
  int spr;             // steps per row = Vq / kStepVec
  int span;            // steps per CTA
  int rpr;             // CTA record blocks per row
  int64_t nsteps;      // B * spr
  const int32_t* slots;
  const sampling_params* params_dev;  // nullable
  const sampling_params* params_tab;
  int pen_mode;
  HistState hs;
  PartRec* parts;      // [B][rpr][kCW]
  RowHand* hand;       // [B]
  PenEnt* pent;        // [B][L]
  uint16_t* gkeys;     // [B][gk_stride(Vq)]: group keys | step keys
  uint64_t* trace;     // debug: per-CTA start / end timestamps (globaltimer ns, 64 per CTA), nullable
  int pen_in_b;        // small batches: phase B builds the hand-off in its prologue (this pass skips it)
  int early_tiles;     // small batches: the first tiles' logits copies before the grid wait
};

// ---- packed binary32 pairs (sm_100a FADD2 / FMUL2) ----------------------------------
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// (lo, hi) bf16 halves of w minus m, each correctly rounded to binary32 (exact when m is a
// bf16 value: the difference of two bf16 numbers fits binary32): fma.rn.f32.bf16(z, 1, -m)
__device__ __forceinline__ uint64_t bf16x2_sub(uint32_t w, float nm) {
  float a, b;
  asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
      "fma.rn.f32.bf16 %0, l, %3, %4;\n\tfma.rn.f32.bf16 %1, h, %3, %4;}"
      : "=f"(a), "=f"(b)
      : "r"(w), "h"((unsigned short)0x3F80), "f"(nm));
  return f2_pack(a, b);
}

// Per-step (group) math.  u = the lane's 4 vectors of the step (masked).  gmax(): NaN-propagating
// max; esum(): sum over the group of 2^((z + nm) * c), nm = -m_ref (the terms of -inf are 0).
template <typename T>
struct GroupMath;
template <>
struct GroupMath<__nv_bfloat16> {
  static __device__ __forceinline__ float gmax(const uint4 (&u)[kG]) {
    __nv_bfloat162 m[4];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u[j].x);
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u[j].y);
      const __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&u[j].z);
      const __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&u[j].w);
      m[j] = __hmax2_nan(__hmax2_nan(a, b), __hmax2_nan(c, d));
    }
    const __nv_bfloat162 r = __hmax2_nan(__hmax2_nan(m[0], m[1]), __hmax2_nan(m[2], m[3]));
    return fmax_nan(__low2float(r), __high2float(r));
  }
  static __device__ __forceinline__ float esum(const uint4 (&u)[kG], float nm, uint64_t c2) {
    float tmax;
    return esum_tmax(u, nm, c2, tmax);
  }
  // the exp-sum and, from the same differences t = z - m_ref (exact for bf16 operands), the
  // NaN-propagating max of t on the FP32 ALU (keeps the packed bf16 max off the MUFU/XU pipe)
  static __device__ __forceinline__ float esum_tmax(const uint4 (&u)[kG], float nm, uint64_t c2, float& tmax) {
    uint64_t e[2 * kG];
    float tm[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
      uint64_t p[4];
      float m4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t t2 = bf16x2_sub(w[i], nm);
        float ta, tb;
        f2_unpack(t2, ta, tb);
        m4[i] = fmax_nan(ta, tb);
        float a, b;
        f2_unpack(f2_mul(t2, c2), a, b);
        p[i] = f2_pack(ex2f(a), ex2f(b));
      }
      tm[j] = fmax_nan(fmax_nan(m4[0], m4[1]), fmax_nan(m4[2], m4[3]));
      e[2 * j] = f2_add(p[0], p[1]);
      e[2 * j + 1] = f2_add(p[2], p[3]);
    }
    tmax = fmax_nan(fmax_nan(tm[0], tm[1]), fmax_nan(tm[2], tm[3]));
#pragma unroll
    for (int s = 1; s < 2 * kG; s <<= 1)
#pragma unroll
      for (int i = 0; i < 2 * kG; i += 2 * s) e[i] = f2_add(e[i], e[i + s]);
    float a, b;
    f2_unpack(e[0], a, b);
    return a + b;
  }
};
template <>
struct GroupMath<float> {
  static __device__ __forceinline__ float gmax(const uint4 (&u)[kG]) {
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kG; ++j) m = fmax_nan(m, Dec<float>::vmax(u[j]));
    return m;
  }
  static __device__ __forceinline__ float esum_tmax(const uint4 (&u)[kG], float nm, uint64_t c2, float& tmax) {
    tmax = gmax(u) + nm;  // (unused for binary32 logits: the max is taken on the raw values)
    return esum(u, nm, c2);
  }
  static __device__ __forceinline__ float esum(const uint4 (&u)[kG], float nm, uint64_t c2) {
    const uint64_t nm2 = f2_pack(nm, nm);
    uint64_t e[2 * kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const uint64_t t0 = f2_add(f2_pack(__uint_as_float(u[j].x), __uint_as_float(u[j].y)), nm2);
      const uint64_t t1 = f2_add(f2_pack(__uint_as_float(u[j].z), __uint_as_float(u[j].w)), nm2);
      float a, b, c, d;
      f2_unpack(f2_mul(t0, c2), a, b);
      f2_unpack(f2_mul(t1, c2), c, d);
      e[2 * j] = f2_pack(ex2f(a), ex2f(b));
      e[2 * j + 1] = f2_pack(ex2f(c), ex2f(d));
    }
#pragma unroll
    for (int s = 1; s < 2 * kG; s <<= 1)
#pragma unroll
      for (int i = 0; i < 2 * kG; i += 2 * s) e[i] = f2_add(e[i], e[i + s]);
    float a, b;
    f2_unpack(e[0], a, b);
    return a + b;
  }
};

// Lane-private online softmax state: acc = sum 2^((z - mref) * c) (float64); a new mref is
// taken when an element exceeds thr = mref + 8 / c.
struct LaneSum {
  float mref, thr, nm, mmax;
  double acc;
  int bad;
  __device__ __forceinline__ void reset() {
    mref = -INFINITY;
    thr = -INFINITY;
    nm = INFINITY;
    mmax = -INFINITY;
    acc = 0.0;
    bad = 0;
  }
  __device__ __forceinline__ void rebase(float m, float c, float inv8) {
    if (acc != 0.0) acc *= (double)ex2f((mref - m) * c);
    mref = m;
    nm = -m;
    thr = m + inv8;
  }
};

template <typename T>
__global__ void __launch_bounds__(kStreamThreads, kStreamCtasPerSm) stream_kernel(const __grid_constant__ StreamArgs a) {
  constexpr int VEC = Dec<T>::N;
  constexpr int ESZ = (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint8_t* ring = smem + kSOffRing;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem + kSOffBm);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSOffBar);
  uint64_t* empty = full + kNS;
  float2* segc = reinterpret_cast<float2*>(smem + kSOffSeg);  // per row of the span: (c, 8 / c)
  const uint4 kNegInfVec = make_uint4(Dec<T>::kNegInfWord, Dec<T>::kNegInfWord, Dec<T>::kNegInfWord,
                                      Dec<T>::kNegInfWord);
  // programmatic dependent launch on both sides: this grid may have been launched while the
  // previous kernel of the stream (the last step's phase B) was still running — wait for it before
  // any memory access (it appends to the histories this pass reads, and reads the scratch this
  // pass writes); then let phase B's CTAs be scheduled as this grid's CTAs retire
  if (!a.early_tiles) {
    griddep_wait();
    griddep_launch();
  }
  const int64_t s0 = (int64_t)blockIdx.x * a.span;
  const int nspan = (int)min((int64_t)a.span, a.nsteps - s0);  // steps of this CTA
  const int ntiles = (nspan + kTileSteps - 1) / kTileSteps;
  const int nvv = (a.vloc + VEC - 1) / VEC;
  const uint8_t* lg = reinterpret_cast<const uint8_t*>(a.logits);
  const int64_t ldb = a.ld * ESZ;
  if (a.trace && tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.trace[blockIdx.x * 64 + 0] = gtimer();
    a.trace[blockIdx.x * 64 + 1] = smid;
  }
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kCW);
    }
    mbar_init(reinterpret_cast<uint64_t*>(smem + kSOffPenBar), 1);
    mbar_init(reinterpret_cast<uint64_t*>(smem + kSOffPenBar) + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // small batches (early_tiles): the first kNS tiles' logits are this call's input, not the last
  // step's output, so their bulk copies are issued before the grid wait (the bitmap words — history
  // state the last step's phase B appends to — after it) and the ring fills while the previous kernel
  // drains (measured: c5 B = 1 19.8 -> 18.8 us; at c3 it costs 0.9 us, so large batches wait first)
  if (a.early_tiles) {
    if (w == kCW && lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      for (int t = 0; t < kNS && t < ntiles; ++t) {
        const int64_t st0 = s0 + (int64_t)t * kTileSteps;
        int r = (int)(st0 / a.spr), k = (int)(st0 - (int64_t)r * a.spr);
        const int n = min(kTileSteps, nspan - t * kTileSteps);
        uint32_t bytes = 0;
        {
          int kk = k;
          for (int j = 0; j < n; ++j) {
            bytes += (uint32_t)min(kStepVec, nvv - kk * kStepVec) * 16u;
            if (++kk == a.spr) kk = 0;
          }
        }
        mbar_arrive_expect_tx(full + t, bytes + (uint32_t)n * 128u);
        uint8_t* dst = ring + t * (kTileSteps * kStepBytes);
        for (int j = 0; j < n;) {
          const int j0 = j, k0 = k;
          uint32_t nb = 0;
          do {
            nb += (uint32_t)min(kStepVec, nvv - k * kStepVec) * 16u;
            ++j;
            ++k;
          } while (j < n && k < a.spr);
          bulk_g2s(dst + j0 * kStepBytes, lg + ((int64_t)r * ldb + (int64_t)k0 * kStepBytes), nb, full + t, pol);
          if (k == a.spr) { k = 0; ++r; }
        }
      }
    }
    griddep_wait();
    griddep_launch();
  }

  if (w == kCW + 1) {
    // ================= penalty warp: the hand-off of the rows that start in this span =================
    const int64_t rfirst = (s0 + a.spr - 1) / a.spr;
    UniqEntry* pbuf = reinterpret_cast<UniqEntry*>(smem + kSOffPen);
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + kSOffPenBar);
    uint32_t pphase[2] = {0u, 0u};
    for (int64_t r = rfirst; !a.pen_in_b && r * a.spr < s0 + nspan; ++r) {
      bool slot_ok;
      const int slot = row_slot(a.slots, (int)r, a.hs.nslots, &slot_ok);
      const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
      const SlotMeta sm = a.hs.meta[slot];
      if (lane == 0) {
        RowHand h;
        h.slot = slot;
        h.pad[0] = slot_ok ? 0 : 1;  // (phase B: SAMPLER_ROW_INVALID)
        h.pad[1] = h.pad[2] = 0;
        h.meta = sm;
        h.prm = prm;
        a.hand[r] = h;
      }
      const UniqEntry* ut = a.hs.uniq + (int64_t)slot * a.hs.L;
      const uint8_t* rowp = lg + r * ldb;
      // batches of kPenB table entries: the table slice bulk-copied into smem (double-buffered: the
      // next batch's copy is in flight while this one's logits are gathered, 32 per lane at once)
      const int nb = (sm.n_uniq + kPenB - 1) / kPenB;
      auto issue = [&](int j) {  // lane 0: batch j into buffer j & 1; returns the 8-byte skew
        const int e0 = j * kPenB, n = min(kPenB, sm.n_uniq - e0);
        const uintptr_t src = reinterpret_cast<uintptr_t>(ut + e0);
        const uintptr_t s16 = src & ~(uintptr_t)15;
        const uint32_t bytes = (uint32_t)(((src - s16) + (uintptr_t)n * 8 + 15) & ~(uintptr_t)15);
        uint64_t* bar = pbar + (j & 1);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s_nohint(pbuf + (j & 1) * (kPenB + 2), reinterpret_cast<const void*>(s16), bytes, bar);
      };
      if (nb > 0 && lane == 0) issue(0);
      for (int j = 0; j < nb; ++j) {
        if (j + 1 < nb && lane == 0) issue(j + 1);  // (its buffer's previous batch is consumed)
        mbar_wait(pbar + (j & 1), pphase[j & 1]);
        pphase[j & 1] ^= 1u;
        const int e0 = j * kPenB, n = min(kPenB, sm.n_uniq - e0);
        const UniqEntry* bu = pbuf + (j & 1) * (kPenB + 2) +
                              ((reinterpret_cast<uintptr_t>(ut + e0) & 15) ? 1 : 0);  // (the skew)
        float raw[kPenB / 32];
#pragma unroll
        for (int q = 0; q < kPenB / 32; ++q) {
          const int e = lane + 32 * q;
          const int le = e < n ? bu[e].id - a.voff : -1;
          raw[q] = (le >= 0 && le < a.vloc) ? Dec<T>::load1(rowp, le) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < kPenB / 32; ++q) {
          const int e = lane + 32 * q;
          if (e >= n) continue;
          const UniqEntry ue = bu[e];
          const int le = ue.id - a.voff;
          PenEnt pe;
          pe.id = ue.id;
          pe.meta = ue.meta;
          pe.zp = (le >= 0 && le < a.vloc) ? apply_penalty(raw[q], ue.meta, prm, a.pen_mode) : 0.f;
          pe.pad = 0;
          a.pent[r * a.hs.L + e0 + e] = pe;
        }
        __syncwarp();  // every lane is done with buffer j & 1 before it is refilled
      }
    }
    if (a.trace && lane == 0) a.trace[blockIdx.x * 64 + 8] = gtimer();
    return;
  }
  if (w == kCW) {
    // ================= producer warp: 1-D bulk copies (TMA engine), one per step =================
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint64_t pwait = 0;
      int r = (int)(s0 / a.spr), k = (int)(s0 - (int64_t)r * a.spr);
      for (int t = 0; t < ntiles; ++t) {
        const int sl = t % kNS;
        const uint64_t tp0 = a.trace ? gtimer() : 0;
        if (t >= kNS) mbar_wait_sleep(empty + sl, (uint32_t)((t / kNS - 1) & 1));
        if (a.trace) pwait += gtimer() - tp0;
        const int n = min(kTileSteps, nspan - t * kTileSteps);
        uint32_t bytes = 0;
        {
          int rr = r, kk = k;
          for (int j = 0; j < n; ++j) {
            bytes += (uint32_t)min(kStepVec, nvv - kk * kStepVec) * 16u;
            if (++kk == a.spr) { kk = 0; ++rr; }
          }
        }
        constexpr bool bmcopy = true;
        const bool early = a.early_tiles && t < kNS;  // (logits already in flight, expect_tx done)
        if (!early) mbar_arrive_expect_tx(full + sl, bytes + (bmcopy ? (uint32_t)n * 128u : 0u));
        uint8_t* dst = ring + sl * (kTileSteps * kStepBytes);
        uint8_t* bdst = reinterpret_cast<uint8_t*>(bm) + sl * (kTileSteps * 128);
        // one bulk copy per run of consecutive steps of one row (contiguous in global memory)
        for (int j = 0; j < n;) {
          const int j0 = j, k0 = k;
          uint32_t nb = 0;
          do {
            nb += (uint32_t)min(kStepVec, nvv - k * kStepVec) * 16u;
            ++j;
            ++k;
          } while (j < n && k < a.spr);
          if (!early)
            bulk_g2s(dst + j0 * kStepBytes, lg + ((int64_t)r * ldb + (int64_t)k0 * kStepBytes), nb, full + sl, pol);
          // the run's penalty-bitmap words (HistState::pmask, 128 B per step)
          if (bmcopy) {
            const int slot = row_slot(a.slots, r, a.hs.nslots, nullptr);
            bulk_g2s(bdst + j0 * 128, a.hs.pmask + ((int64_t)slot * a.spr + k0) * 32, (uint32_t)(j - j0) * 128u,
                     full + sl, pol);
          }
          if (k == a.spr) { k = 0; ++r; }
        }
      }
      if (a.trace) {
        a.trace[blockIdx.x * 64 + 9] = pwait;
        a.trace[blockIdx.x * 64 + 10] = gtimer();
      }
    }
    return;
  }

  // ================= consumer warps =================
  // span rows: constants, and every (row, this CTA, warp) partial record initialised empty
  const int r_cta0 = (int)(s0 / a.spr);
  const int r_cta1 = (int)((s0 + nspan - 1) / a.spr);
  for (int g = w; g <= r_cta1 - r_cta0; g += kCW) {
    const int r = r_cta0 + g;
    const int slot = row_slot(a.slots, r, a.hs.nslots, nullptr);
    const sampling_params* gprm = a.params_dev ? a.params_dev + r : a.params_tab + slot;
    const float temp = gprm->temperature;
    const float tau = (temp < kGreedyEps) ? 1.0f : temp;
    const float c = __fdiv_rn((float)kLog2e, tau);
    if (lane == 0) segc[g] = make_float2(c, __fdiv_rn(8.0f, c));
    const int64_t cfirst = ((int64_t)r * a.spr) / a.span;
    if (lane < kCW) {
      PartRec pr;
      pr.m = -INFINITY;
      pr.bad = 0u;
      pr.s = 0.0;
      a.parts[((int64_t)r * a.rpr + (blockIdx.x - cfirst)) * kCW + lane] = pr;
    }
  }
  cbar_n<kCW * 32>();  // the span's row constants are in smem

  int cur = -1;  // row being accumulated
  LaneSum ls;
  ls.reset();
  float c = 0.f, inv8 = 0.f;
  uint64_t c2 = 0;
  uint16_t* gkr = nullptr;
  auto flush = [&]() {
    const float m = warp_max(ls.mmax);
    double sv = (ls.acc != 0.0) ? ls.acc * (double)ex2f((ls.mref - m) * c) : 0.0;
    sv = warp_sum_d(sv);
    const int bad = __any_sync(kFull, ls.bad);
    if (lane == 0) {
      const int64_t cfirst = ((int64_t)cur * a.spr) / a.span;
      PartRec pr;
      pr.m = m;
      pr.bad = bad ? kRecBad : 0u;
      pr.s = sv;
      a.parts[((int64_t)cur * a.rpr + (blockIdx.x - cfirst)) * kCW + w] = pr;
    }
  };
  // this warp's step cursor: CTA-relative step i = 16 t + w  <->  (row r, row step k)
  int r = (int)((s0 + w) / a.spr), k = (int)(s0 + w - (int64_t)r * a.spr);
  for (int t = 0; t < ntiles; ++t) {
    const int i = t * kTileSteps + w;
    const int sl = t % kNS;
    if (i < nspan) {
      if (r != cur) {
        if (cur >= 0) flush();
        cur = r;
        const float2 cc = segc[r - r_cta0];
        c = cc.x;
        inv8 = cc.y;
        c2 = f2_pack(c, c);
        ls.reset();
        gkr = a.gkeys + (int64_t)r * gk_stride(a.Vq);
      }
      const int vb = k * kStepVec;
      uint4 cur4[kG];
      __syncwarp();  // converged before the spin-wait (a diverged lane must not starve behind it)
      mbar_wait_sleep(full + sl, (uint32_t)((t / kNS) & 1));
      const uint4* tile = reinterpret_cast<const uint4*>(ring + sl * (kTileSteps * kStepBytes) + w * kStepBytes);
      uint32_t pm = bm[(sl * kTileSteps + w) * 32 + lane];
      if (vb + kStepVec <= nvv) {
#pragma unroll
        for (int j = 0; j < kG; ++j) cur4[j] = tile[lane + 32 * j];
      } else {  // the row's last (partial) step: past the row -inf, the padding tail masked
#pragma unroll
        for (int j = 0; j < kG; ++j) cur4[j] = (vb + lane + 32 * j < nvv) ? tile[lane + 32 * j] : kNegInfVec;
#pragma unroll
        for (int j = 0; j < kG; ++j)
#pragma unroll
          for (int tt = 0; tt < VEC; ++tt)
            if ((vb + lane + 32 * j) * VEC + tt >= a.vloc) pm |= 1u << (j * VEC + tt);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + sl);  // this warp's part of the slot is consumed
      if (pm) {
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          const uint32_t b = (pm >> (j * VEC)) & ((1u << VEC) - 1u);
          if (b) cur4[j] = Dec<T>::mask(cur4[j], b);
        }
      }
      // The lane's first finite group takes its max as the reference (the only place the max is
      // taken separately); afterwards one exp-sum pass per group also yields the group max (bf16:
      // from the exact differences t = z - m_ref).  A group exceeding the reference by > 8 / c
      // (rare) rebases and runs the same pass again — one copy of the pass in the loop.
      float gm = -INFINITY, es = 0.f;
      if (!(ls.mref > -INFINITY)) {
        const float g0 = GroupMath<T>::gmax(cur4);
        if (g0 > -INFINITY) ls.rebase(g0, c, inv8);
        gm = g0;  // (stays -inf / NaN when the group has no finite element)
      }
      if (ls.mref > -INFINITY) {
        for (;;) {
          float tmax;
          es = GroupMath<T>::esum_tmax(cur4, ls.nm, c2, tmax);
          // bf16: t = z - m_ref is exact (and so is t + m_ref = z) when |m_ref| < 2^16 |z|; otherwise
          // (a group far below the reference) the max is taken on the raw values
          gm = (VEC == 8) ? tmax + ls.mref : GroupMath<T>::gmax(cur4);
          if (VEC == 8 && !(fabsf(ls.mref) <= 16384.0f * fabsf(gm))) gm = GroupMath<T>::gmax(cur4);
          if (!(gm > ls.thr)) break;
          ls.rebase(gm, c, inv8);
        }
      }
      ls.bad |= !(gm < INFINITY) ? 1 : 0;  // NaN or +inf in the group
      uint32_t key;
      if (VEC == 8) {  // bf16 logits: gm is a bf16 value, its key is its bits, order-flipped
        const uint32_t h = __float_as_uint(gm + 0.0f) >> 16;  // (-0 -> +0)
        key = (gm != gm) ? 0xFF80u : h ^ ((h & 0x8000u) ? 0xFFFFu : 0x8000u);  // NaN: the +inf key
      } else {
        key = key16_down(gm);
      }
      gkr[k * 32 + lane] = (uint16_t)key;
      const uint32_t skey = __reduce_max_sync(kFull, key);
      if (lane == 0) gkr[a.Vq / kG + k] = (uint16_t)skey;
      if (gm > -INFINITY) {
        ls.acc += (double)es;
        ls.mmax = fmaxf(ls.mmax, gm);
      }
    } else if (lane == 0) {
      mbar_arrive(empty + sl);
    }
    k += kTileSteps;
    while (k >= a.spr) {
      k -= a.spr;
      ++r;
    }
  }
  if (cur >= 0) flush();
  if (a.trace && tid == 0) a.trace[blockIdx.x * 64 + 7] = gtimer();
}

}  // namespace smp

// select.cuh — phase B of the sampling step: one CTA per row turns the row's piece records and
// group keys (phase A, stream.cuh) into the exact top-K candidates and the sample.
//
// One dependent chain per row, shaped for latency (the GPU is otherwise idle while it runs):
//   prologue   (independent of phase A; overlaps its tail under programmatic dependent launch)
//              the slot's unique-token table -> smem, raw logits of its ids -> registers
//   RT1        piece headers and the row's group keys (one round trip); M, S from the headers
//   bound      T = K-th largest 16-bit key among the group keys and the penalised elements: one
//              smem histogram over the kHistBins key steps below key(M) (one bin per key value,
//              so T is exact).  K distinct elements are >= val(T)
//   collect    penalised ids: exact penalised value from the prefetched raws;
//              groups with key >= key(T): re-read (RT2), penalised ids and padding masked, every
//              element >= T pushed — the pool then holds EVERY element of the row >= T, exactly
//   top-K      rank counting over the pool (exact, ties impossible: composites are unique)
//   decide     warp 0 (merge.cuh warp_decide): top-k -> top-p -> min-p, Philox draw in id order
//   append     the sampled token into the slot's history (block-parallel shift from the smem copy)
// mode 1 (vocab-sharded phase 1) emits the row's candidate record instead of deciding.
#pragma once
#include <cfloat>
#include "block.cuh"
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "philox.cuh"
#include "piece.cuh"
#include "stream.cuh"

namespace smp {

constexpr int kSelPen = 2048;          // unique-token entries staged in smem
constexpr int kSelSpec = 1024;         // penalised entries loaded speculatively in RT1 (the rest, if
                                       // n_uniq is larger, after the hand-off arrives)
constexpr int kSelPR = kSelSpec / kBT;  // per thread
constexpr int kSelQ = 2048;            // qualifying-group list capacity
constexpr int kSelGR = 3;              // group-key words (8 keys) per thread per chunk

struct SelectArgs {
  const void* logits;
  int64_t ld;
  int B, V, voff, vloc;
  int64_t Vq;
  int spr, span, rpr;  // phase A geometry (stream.cuh)
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  const uint64_t* step_dev;  // nullable: the decode step read on the device
  int kcand, pen_mode, mode, append, pending_ok;
  HistState hs;
  const PartRec* parts;    // phase A partial records [B][rpr][kCW]
  const RowHand* hand;     // phase A hand-off [B]
  const PenEnt* pent;      // [B][L]
  const uint16_t* gkeys;
  RowOut ro;
  uint8_t* out_records;  // mode 1: one candidate record per row
  int64_t out_stride;
  ExchPeers xp;          // mode 1 with xp.world > 0: records stored into every peer (NEXT-2)
  int fuse_merge;        // with xp: this CTA then waits for every rank's record of its row and merges
                         // them (outputs in ro, append) — the exchange and the merge in one kernel
  int pen_in_b;          // small batches: the row's hand-off is built here, before the grid wait
  uint64_t* trace;       // debug: per-row phase timestamps (32 per row), nullable
};

// shared-memory carve-up (phase B)
constexpr int kSOffUe = 0;                                         // [kSelPen] UniqEntry
constexpr int kHistBins = 1024;                                    // bound histogram (key steps)
constexpr int kSOffHist = kSOffUe + kSelPen * 8;                   // [kHistBins] u32
constexpr int kSOffPool = kSOffHist + kHistBins * 4;               // [kPool] u64
constexpr int kSOffQl = kSOffPool + kPool * 8;                     // [kSelQ] u32
constexpr int kSOffTop = kSOffQl + kSelQ * 4;                      // [KC] u64
constexpr int kSOffWv = kSOffTop + SAMPLER_KCAND_MAX * 8;          // [KC] double
constexpr int kSOffById = kSOffWv + SAMPLER_KCAND_MAX * 8;         // [KC] u64
constexpr int kSOffHdr = kSOffById + SAMPLER_KCAND_MAX * 8;        // [kMaxRecW] RecHdr
constexpr int kSOffScr = kSOffHdr + kMaxRecW * 48;                 // f[8] d[8] u[16] i[16]
constexpr int kSOffCtl = kSOffScr + 288;                           // ints [16]
constexpr int kSOffGk = kSOffCtl + 64;                             // [kSelGR * kBT] uint4 group keys
constexpr int kSOffSk = kSOffGk + kSelGR * kBT * 16;               // [kBT] u16 step keys
constexpr int kSOffHand = kSOffSk + kBT * 2;                        // RowHand
constexpr int kSOffZp = kSOffHand + (int)sizeof(RowHand);          // [kSelPen] float penalised values
constexpr int kSelectSmem = kSOffZp + kSelPen * 4;


// Append `tok` to the slot's history (P:371 incremental update) from the smem copy of the sorted
// unique-token table s_ue[0..nu) (nu <= kSelPen): the insertion point by binary search, then every
// entry above it is stored one slot up straight from smem.
__device__ __forceinline__ void block_append_smem(const HistState& hs, int slot, int32_t tok, const SlotMeta& sm,
                                                  const UniqEntry* s_ue, const BlockScratch& bs) {
  const int tid = threadIdx.x;
  const int nu = sm.n_uniq, np = sm.n_prompt, no = sm.n_out;
  if (np + no + 1 > hs.L) {
    if (tid == 0) hs.meta[slot].flags |= 1;
    return;
  }
  // insertion point by binary search of the id-sorted table, in every thread (smem broadcasts,
  // no block barrier)
  int lo = 0, hi = nu;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_ue[mid].id < tok) lo = mid + 1;
    else hi = mid;
  }
  const int less = lo;
  const bool found = less < nu && s_ue[less].id == tok;
  UniqEntry* u = hs.uniq + (int64_t)slot * hs.L;
  if (found) {
    if (tid == 0) u[less].meta = s_ue[less].meta + 2u;
  } else {
    for (int i = less + tid; i < nu; i += kBT) u[i + 1] = s_ue[i];
    if (tid == 0) {
      UniqEntry e;
      e.id = tok;
      e.meta = 2u;
      u[less] = e;
    }
    if (tid == 0) pmask_set(hs, slot, tok);
  }
  if (tid == 0) {
    hs.tokens[(int64_t)slot * hs.L + np + no] = tok;
    SlotMeta m2 = sm;
    m2.n_out = no + 1;
    if (!found) m2.n_uniq = nu + 1;
    hs.meta[slot] = m2;
  }
}

// Degenerate rows (more candidates >= T than the pool holds: massive ties, or an unbounded T):
// the whole collection again in bounded chunks, shrinking the pool to its exact top-K (raising a
// floor below which nothing is kept) whenever it fills.  Returns the floor.
// float64 exp2 / exp / log as calls: one copy of the math-library code on the per-row path
// (each CTA walks its code once, so inlined copies are instruction-fetch misses)
__device__ __noinline__ double dexp2_call(double x) { return exp2(x); }
__device__ __noinline__ double dexp_call(double x) { return exp(x); }
__device__ __noinline__ double dlog_call(double x) { return log(x); }

template <typename T>
__device__ __noinline__ uint64_t select_collect_slow(const SelectArgs& a, const uint8_t* rowp,
                                                    const UniqEntry* utab, const UniqEntry* s_ue, int nu, int nus,
                                                    const sampling_params& prm, float Tv, uint32_t lo_k, int nvv,
                                                    int gwords, int keff, const MergeSmem& ms, int* ctl,
                                                    uint32_t* hist) {
  constexpr int VEC = Dec<T>::N;
  const int tid = threadIdx.x;
  uint64_t floor = 0;
  cbar();
  if (tid == 0) ctl[1] = 0;
  cbar();
  auto push = [&](uint64_t c) {
    if (c < floor) return;
    const int at = atomicAdd(&ctl[1], 1);
    if (at < kPool) ms.pool[at] = c;
  };
  auto shrink = [&]() {  // uniform: after a barrier
    const int cnt = ctl[1];
    if (cnt > kPool - 1024) {
      const uint64_t Tc = block_kth_largest(ms.pool, cnt, keff, hist, ms.bs);
      uint64_t kmin;
      const int nn = block_compact_ge(ms.pool, cnt, Tc, &ctl[4], ms.bs, &kmin);
      floor = Tc > floor ? Tc : floor;
      if (tid == 0) ctl[1] = nn;
      cbar();
    }
  };
  for (int e0 = 0; e0 < nu; e0 += kBT) {
    const int e = e0 + tid;
    if (e < nu) {
      const UniqEntry ue = (e < nus) ? s_ue[e] : utab[e];
      const int l = ue.id - a.voff;
      if (l >= 0 && l < a.vloc) {
        const float zp = apply_penalty(Dec<T>::load1(rowp, l), ue.meta, prm, a.pen_mode);
        if (zp >= Tv && zp > -INFINITY && zp < INFINITY) push(make_comp(zp, ue.id));
      }
    }
    cbar();
    shrink();
  }
  const uint16_t* gk = a.gkeys + (int64_t)blockIdx.x * gk_stride(a.Vq);
  for (int g0 = 0; g0 < gwords * 8; g0 += 32) {  // 32 groups = 128 vectors per round
    if (tid < 128) {
      const int g = g0 + (tid >> 2);
      const int v = (g >> 5) * kStepVec + (g & 31) + 32 * (tid & 3);
      if (gk[g] >= lo_k && v < nvv) {
        uint4 u4 = ldg_stream(rowp + (int64_t)v * 16);
        uint32_t msk = listed_mask<VEC>(s_ue, nus, a.voff + v * VEC);
        for (int e = nus; e < nu; ++e) {
          const int k = utab[e].id - a.voff - v * VEC;
          if (k >= 0 && k < VEC) msk |= 1u << k;
        }
#pragma unroll
        for (int t = 0; t < VEC; ++t)
          if (v * VEC + t >= a.vloc) msk |= 1u << t;
        if (msk) u4 = Dec<T>::mask(u4, msk);
#pragma unroll
        for (int t = 0; t < VEC; ++t) {
          const float z = Dec<T>::elem(u4, t);
          if (z >= Tv && z > -INFINITY && z < INFINITY) push(make_comp(z, a.voff + v * VEC + t));
        }
      }
    }
    cbar();
    shrink();
  }
  return floor;
}


// Final decision for one row by the whole block, candidate-parallel (R6-R11; the same
// rules as merge.cuh warp_decide): candidate i = top[i] (pi order, weight wv[i] = exp((z'-M)/tau)
// in float64) is owned by thread i.  Every prefix sum is a fixed-order warp scan plus the warp totals (pi order
// for top-k/top-p, ascending id for the draw), so the arithmetic is the oracle's sequential sums
// (deterministic).  Returns the token (-1: not OK).
__device__ __forceinline__ int block_decide(const MergeSmem& ms, int* ctl, int n, float M, double S, double logS,
                                         uint64_t F, bool bad, bool invalid, const RowCfg& rc, const sampling_params& p,
                                         double u, int row, const RowOut& ro, bool pending_ok, uint64_t* tr) {
  constexpr int UNK = 0x7FFFFFFF;
#define BTR(k)                                    \
  do {                                            \
    if (tr && threadIdx.x == 0) tr[k] = gtimer(); \
  } while (0)
  BTR(8);
  const int tid = threadIdx.x;
  const uint64_t* top = ms.top;
  const double* wv = ms.wv;
  // ctl[6] n2 (top-p), ctl[7] nm (min-p), ctl[8] pick id, ctl[9] n_exact
  if (tid == 0) {
    ctl[6] = UNK;
    ctl[7] = UNK;
    ctl[8] = UNK;
    ctl[9] = 0;
  }
  cbar();
  int status = SAMPLER_ROW_OK;
  if (invalid) status = SAMPLER_ROW_INVALID;
  else if (bad) status = SAMPLER_ROW_NONFINITE;
  else if (n == 0 || !(M > -INFINITY)) status = SAMPLER_ROW_ALL_NEG_INF;
  // n_exact = |{i : top[i] >= F}| (a prefix: top is sorted descending)
  const bool own = tid < n;
  const uint64_t ci = own ? top[tid] : 0ull;
  const double wi = own ? wv[tid] : 0.0;
  if (own && ci >= F && (tid + 1 == n || top[tid + 1] < F)) ctl[9] = tid + 1;
  const bool complete = (F == 0);
  // inclusive pi-order prefix of the weights: warp scans + the totals of the warps before
  const int lane = tid & 31, wq = tid >> 5;
  double cum = warp_incl_scan_d((own && status == SAMPLER_ROW_OK && !rc.greedy) ? wi : 0.0, lane);
  if (lane == 31) ms.bs.d[wq] = cum;
  cbar();
  for (int j = 0; j < wq; ++j) cum += ms.bs.d[j];
  BTR(9);
  const int n_exact = ctl[9];
  int n3 = -1;
  int32_t tok = -1;
  double lp = NAN, flp = NAN, W = 0.0;
  uint64_t cutoff = 0;
  if (status == SAMPLER_ROW_OK) {
    if (rc.greedy) {
      n3 = (n_exact >= 1) ? 1 : -1;
    } else {
      int n1 = UNK;
      if (rc.topk_on) {
        if (rc.k <= n_exact) n1 = rc.k;
        else if (complete) n1 = n;
      } else if (complete) {
        n1 = n;
      }
      int cand = n1;
      bool ok = true;
      double* cums = reinterpret_cast<double*>(ms.pool);  // pi-order prefix sums (the pool is done)
      if (own) cums[tid] = cum;
      cbar();
      if (rc.top_p < 1.0f) {
        double W1 = 0.0;
        bool w1k = false;
        if (n1 != UNK) {
          W1 = cums[n1 - 1];
          w1k = true;
        } else if (!rc.topk_on) {
          W1 = S;
          w1k = true;
        }
        if (!w1k) {
          ok = false;
        } else {
          const double target = (double)rc.top_p * W1;
          const int lim = (n1 != UNK && n1 < n_exact) ? n1 : n_exact;
          if (tid < lim && cum >= target && (tid == 0 || cums[tid - 1] < target)) ctl[6] = tid + 1;
          cbar();
          int n2 = ctl[6];
          if (n2 == UNK && n1 != UNK && n1 <= n_exact) n2 = n1;  // rounding shortfall
          if (n2 != UNK) cand = cand < n2 ? cand : n2;
        }
      }
      if (ok && rc.min_p > 0.0f) {
        if (tid < n_exact && wi < (double)rc.min_p && (tid == 0 || wv[tid - 1] >= (double)rc.min_p)) ctl[7] = tid;
        cbar();
        int nm = ctl[7];
        if (nm == UNK && complete) nm = n;
        if (nm != UNK) cand = cand < nm ? cand : nm;
      }
      if (ok && cand != UNK && cand <= n_exact && cand >= 1) n3 = cand;
      if (n3 >= 1) W = cums[n3 - 1];
    }
    BTR(10);
    if (n3 < 0) {
      status = kRowPending;
    } else {
      cutoff = top[n3 - 1];
      if (rc.greedy) {
        tok = comp_id(top[0]);
        W = 1.0;
        lp = ((double)comp_val(top[0]) - (double)M) - logS;
        flp = 0.0;
      } else {
        // the draw: ascending token id over the kept set K3 = top[0..n3), first cumulative > u W
        const double target = u * W;
        // id order: every kept candidate's rank by id (independent compares), its weight placed
        // at that rank, one scan, the first rank whose cumulative mass exceeds u W
        const int idi = own ? comp_id(ci) : 0;
        double* wid = reinterpret_cast<double*>(ms.byid);     // [n3] weights in id order
        int* idord = reinterpret_cast<int*>(ms.pool + 1024);  // [n3] ids in id order
        if (tid < n3) {
          int rk = 0;
          for (int j = 0; j < n3; ++j) rk += (comp_id(top[j]) < idi) ? 1 : 0;
          wid[rk] = wi;
          idord[rk] = idi;
        }
        cbar();
        double ci_ = warp_incl_scan_d((tid < n3) ? wid[tid] : 0.0, lane);
        if (lane == 31) ms.bs.d[wq] = ci_;
        cbar();
        double off = 0.0;
        for (int j = 0; j < wq; ++j) off += ms.bs.d[j];
        const double prev = __shfl_up_sync(kFull, ci_, 1);
        ci_ += off;
        const double cprev = (lane == 0) ? off : prev + off;
        if (tid < n3 && ci_ > target && !(cprev > target)) ctl[8] = idord[tid];
        cbar();
        BTR(11);
        int pick = ctl[8];
        if (pick == UNK) pick = idord[n3 - 1];  // u W at the top of the mass: the last kept id
        tok = pick;
        if (tid < n3 && idi == pick) {
          lp = ((double)comp_val(ci) - (double)M) / (double)rc.tau - logS;
          flp = dlog_call(wi / W);
          ro.logprobs[row] = (float)lp;
          if (ro.flogprobs) ro.flogprobs[row] = (float)flp;
        }
      }
    }
  }
  BTR(12);
  if (tid == 0) {
    RowInfo ri;
    ri.M = M;
    ri.status = status;
    ri.S = S;
    ri.W = W;
    ri.cutoff = cutoff;
    ri.token = tok;
    ri.greedy = rc.greedy;
    ro.info[row] = ri;
    const bool pend = status == kRowPending;
    if (!pend || !pending_ok) {
      const int st = pend ? SAMPLER_ROW_UNRESOLVED : status;
      ro.tokens[row] = (st == SAMPLER_ROW_OK) ? tok : -1;
      if (st != SAMPLER_ROW_OK || rc.greedy) {
        ro.logprobs[row] = (st == SAMPLER_ROW_OK) ? (float)lp : NAN;
        if (ro.flogprobs) ro.flogprobs[row] = (st == SAMPLER_ROW_OK) ? (float)flp : NAN;
      }
      if (ro.status) ro.status[row] = st;
    }
  }
  BTR(13);
#undef BTR
  return (status == SAMPLER_ROW_OK) ? tok : -1;
}

template <typename T>
__global__ void __launch_bounds__(kBT, 2) select_rows_kernel(const __grid_constant__ SelectArgs a) {
  constexpr int VEC = Dec<T>::N;
  constexpr int ESZ = (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  const int r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  UniqEntry* s_ue = reinterpret_cast<UniqEntry*>(smem + kSOffUe);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + kSOffHist);
  int* ctl = reinterpret_cast<int*>(smem + kSOffCtl);  // [0] T key [1] pool count [2] group count
  MergeSmem ms;
  ms.pool = reinterpret_cast<uint64_t*>(smem + kSOffPool);
  ms.top = reinterpret_cast<uint64_t*>(smem + kSOffTop);
  ms.wv = reinterpret_cast<double*>(smem + kSOffWv);
  ms.byid = reinterpret_cast<uint64_t*>(smem + kSOffById);
  ms.hdr = reinterpret_cast<RecHdr*>(smem + kSOffHdr);
  ms.off = nullptr;
  ms.bs.f = reinterpret_cast<float*>(smem + kSOffScr);
  ms.bs.d = reinterpret_cast<double*>(smem + kSOffScr + 32);
  ms.bs.u = reinterpret_cast<uint64_t*>(smem + kSOffScr + 96);
  ms.bs.i = reinterpret_cast<int*>(smem + kSOffScr + 224);
  uint32_t* ql = reinterpret_cast<uint32_t*>(smem + kSOffQl);
  uint64_t* tr = a.trace ? a.trace + 32 * (int64_t)r : nullptr;
#define STR(k)                                           \
  do {                                                   \
    if (tr && threadIdx.x == 0) tr[k] = gtimer();        \
  } while (0)
  STR(0);

  if (tid == 0) {
    ctl[0] = 0;
    ctl[1] = 0;
    ctl[2] = 0;
    ctl[5] = 0;
  }
  if (a.pen_in_b) {
    // small batches (phase A leaves SMs free, so this prologue overlaps it): the row's hand-off —
    // slot, meta, params and every history entry's exact penalised logit — from the
    // inputs alone (the last step's appends completed before phase A started)
    bool slot_ok;
    const int slot = row_slot(a.slots, r, a.hs.nslots, &slot_ok);
    const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
    const SlotMeta sm0 = a.hs.meta[slot];
    if (tid == 0) {
      RowHand h;
      h.slot = slot;
      h.pad[0] = slot_ok ? 0 : 1;
      h.pad[1] = h.pad[2] = 0;
      h.meta = sm0;
      h.prm = prm;
      const_cast<RowHand*>(a.hand)[r] = h;
    }
    const UniqEntry* ut = a.hs.uniq + (int64_t)slot * a.hs.L;
    const uint8_t* rp = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * ESZ;
    PenEnt* pe = const_cast<PenEnt*>(a.pent) + (int64_t)r * a.hs.L;
#pragma unroll 1
    for (int e0 = 0; e0 < sm0.n_uniq; e0 += 4 * kBT) {
      UniqEntry ue[4];
      float raw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * kBT + tid;
        if (e < sm0.n_uniq) ue[q] = ut[e];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * kBT + tid;
        const int le = e < sm0.n_uniq ? ue[q].id - a.voff : -1;
        raw[q] = (le >= 0 && le < a.vloc) ? Dec<T>::load1(rp, le) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * kBT + tid;
        if (e >= sm0.n_uniq) continue;
        const int le = ue[q].id - a.voff;
        PenEnt x;
        x.id = ue[q].id;
        x.meta = ue[q].meta;
        x.zp = (le >= 0 && le < a.vloc) ? apply_penalty(raw[q], ue[q].meta, prm, a.pen_mode) : 0.f;
        x.pad = 0;
        pe[e] = x;
      }
    }
    cbar();
  }
  griddep_wait();  // phase A's hand-off, partial records and keys are visible from here on
  griddep_launch();  // the next step's phase A may be scheduled as these CTAs retire (it waits)
  // ---- RT1 (one round trip, nothing indexed by slot): the hand-off, the penalised entries, the
  // partial records, the step keys and the group keys of row r
  RowHand* s_hand = reinterpret_cast<RowHand*>(smem + kSOffHand);
  if (tid < (int)(sizeof(RowHand) / 16))
    reinterpret_cast<uint4*>(s_hand)[tid] = reinterpret_cast<const uint4*>(a.hand + r)[tid];
  const int ncap = min(a.hs.L, kSelSpec);  // entries loaded speculatively (nu is in the hand-off)
  float* s_zp = reinterpret_cast<float*>(smem + kSOffZp);
  {
    uint4 x[kSelPR];  // every load in flight before the first use
    const uint4* src = reinterpret_cast<const uint4*>(a.pent + (int64_t)r * a.hs.L);
#pragma unroll
    for (int q = 0; q < kSelPR; ++q)
      if (tid + q * kBT < ncap) x[q] = src[tid + q * kBT];
#pragma unroll
    for (int q = 0; q < kSelPR; ++q) {
      const int e = tid + q * kBT;
      if (e < ncap) {
        UniqEntry ue;
        ue.id = (int32_t)x[q].x;
        ue.meta = x[q].y;
        s_ue[e] = ue;
        s_zp[e] = __uint_as_float(x[q].z);
      }
    }
  }
  const int64_t cfirst = ((int64_t)r * a.spr) / a.span;
  const int64_t clast = ((int64_t)(r + 1) * a.spr - 1) / a.span;
  const int nparts = (int)(clast - cfirst + 1) * kCW;
  const PartRec* prow = a.parts + (int64_t)r * a.rpr * kCW;
  PartRec p0;
  p0.m = -INFINITY;
  p0.bad = 0u;
  p0.s = 0.0;
  if (tid < nparts) p0 = prow[tid];
  const int nvv = (a.vloc + VEC - 1) / VEC;
  const int gwords = ((nvv + kStepVec - 1) / kStepVec) * 32 / 8;  // valid group-key words (8 keys)
  const uint4* gk4 = reinterpret_cast<const uint4*>(a.gkeys + (int64_t)r * gk_stride(a.Vq));
  const uint16_t* sk = a.gkeys + (int64_t)r * gk_stride(a.Vq) + a.Vq / kG;  // step keys
  const int nsv = (nvv + kStepVec - 1) / kStepVec;                             // real steps
  uint16_t* s_sk = reinterpret_cast<uint16_t*>(smem + kSOffSk);
  if (tid < nsv && tid < kBT) s_sk[tid] = sk[tid];
  uint4* s_gk = reinterpret_cast<uint4*>(smem + kSOffGk);
#pragma unroll
  for (int q = 0; q < kSelGR; ++q) {  // staged in smem: every load of RT1 completes at one barrier
    const int w = tid + q * kBT;
    s_gk[w] = (w < gwords) ? gk4[w] : make_uint4(0, 0, 0, 0);
  }
  for (int i = tid; i < kHistBins; i += kBT) hist[i] = 0u;
  cbar();
  const int slot = s_hand->slot;
  const sampling_params prm = a.params_dev ? a.params_dev[r] : s_hand->prm;
  // device-supplied slots / params are validated here (SAMPLER_ROW_INVALID; the slot is not touched)
  const bool invalid = s_hand->pad[0] != 0 || !params_ok(prm, a.pen_mode);
  const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
  const RowCfg rc = decode_row(prm, a.V, a.kcand);
  const int keff = rc.keff;
  const SlotMeta smeta = s_hand->meta;
  const int nu = smeta.n_uniq;
  const int nus = min(nu, kSelPen);
  if (nus > ncap) {  // (uniform) a long history: the rest of the smem-staged entries
    const uint4* src = reinterpret_cast<const uint4*>(a.pent + (int64_t)r * a.hs.L);
    for (int e = ncap + tid; e < nus; e += kBT) {
      const uint4 x = src[e];
      UniqEntry ue;
      ue.id = (int32_t)x.x;
      ue.meta = x.y;
      s_ue[e] = ue;
      s_zp[e] = __uint_as_float(x.z);
    }
    cbar();
  }
  const UniqEntry* utab = a.hs.uniq + (int64_t)slot * a.hs.L;
  const uint8_t* rowp = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * ESZ;
  // very long tables (nu > kSelPen): the entries past the smem copy straight from phase A's hand-off
  // (id, meta, exact z'), 4 per thread in flight; fn(id, local id, z') for those inside the slice
  const uint4* pent_r = reinterpret_cast<const uint4*>(a.pent + (int64_t)r * a.hs.L);
  auto for_long = [&](auto&& fn) {
#pragma unroll 1
    for (int e0 = kSelPen + tid; e0 < nu; e0 += 4 * kBT) {
      uint4 x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e0 + q * kBT < nu) x[q] = pent_r[e0 + q * kBT];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (e0 + q * kBT >= nu) break;
        const int l = (int)x[q].x - a.voff;
        if (l >= 0 && l < a.vloc) fn((int)x[q].x, l, __uint_as_float(x[q].z));
      }
    }
  };
  // the penalised entries: smem copy of the table (id order) for masking and the append, and the
  // exact penalised values s_zp (entries outside this vocabulary slice are skipped by id)
  STR(1);
  // ---- M = max of the stream partials and the exact penalised values;
  //      S = sum_parts s 2^((m - M) c) + sum_pen 2^((z' - M) c)   (fixed order: deterministic)
  float mloc = p0.m;
  unsigned fl = p0.bad;
  for (int o = tid + kBT; o < nparts; o += kBT) {
    const PartRec pr = prow[o];
    mloc = fmaxf(mloc, pr.m);
    fl |= pr.bad;
  }
#pragma unroll 1
  for (int e = tid; e < nus; e += kBT) {
    const int l = s_ue[e].id - a.voff;
    if (l < 0 || l >= a.vloc) continue;
    const float zp = s_zp[e];
    if (!(zp < INFINITY)) fl |= kRecBad;  // NaN / +inf logit (or penalised value)
    else mloc = fmaxf(mloc, zp);
  }
  for_long([&](int, int, float zp) {
    if (!(zp < INFINITY)) fl |= kRecBad;
    else mloc = fmaxf(mloc, zp);
  });
  // one barrier for max and flags together; meanwhile the last warp finds the bound T = the K-th
  // largest step key (each step key = the max of 1024 / 512 elements rounded down, so K distinct
  // elements are >= val(T); every element >= val(T) lies in a group with key >= T or is
  // penalised): warp radix select, MSB first — the largest x with |{step keys >= x}| >= K
  {
    const int w = tid >> 5;
    float mw = warp_max(mloc);
    const unsigned fw = __reduce_or_sync(kFull, fl);
    if (lane == 0) {
      ms.bs.f[w] = mw;
      ms.bs.i[w] = (int)fw;
    }
    if (w == kBW - 2 && lane == 0) {  // the draw's uniform, off the critical path
      const double uu = philox_uniform(seed, prm.request_id, a.step_dev ? *a.step_dev : a.step);
      *reinterpret_cast<double*>(ctl + 14) = uu;
    }
    if (w == kBW - 1 && nsv >= keff && nsv <= kBT) {
      uint32_t key[8];  // 8 keys per lane at most: nsv <= 256
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = lane + 32 * i;
        const uint32_t y = (j < nsv) ? (uint32_t)s_sk[j] : 0u;
        key[i] = (y > kKey16NegInf) ? y : 0u;
      }
      uint32_t pre = 0;
#pragma unroll 1
      for (int b = 15; b >= 0; --b) {
        const uint32_t cand = pre | (1u << b);
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) cnt += __popc(__ballot_sync(kFull, key[i] >= cand));
        if (cnt >= keff) pre = cand;
      }
      if (lane == 0 && pre > kKey16NegInf) ctl[0] = (int)pre;  // (fewer than K finite keys: 0)
    }
    cbar();
    mw = ms.bs.f[0];
    unsigned fa = (unsigned)ms.bs.i[0];
#pragma unroll
    for (int j = 1; j < kBW; ++j) {
      mw = fmaxf(mw, ms.bs.f[j]);
      fa |= (unsigned)ms.bs.i[j];
    }
    mloc = mw;
    fl = fa;
  }
  const float M = mloc;
  const bool bad = (fl & kRecBad) != 0;
  STR(2);
  double term = 0.0;
  auto s_terms = [&]() -> double {
    double t = 0.0;
    if (!(M > -INFINITY) || bad) return t;
    if (p0.s != 0.0) t += p0.s * dexp2_call(((double)p0.m - (double)M) * rc.c_d);
#pragma unroll 1
    for (int o = tid + kBT; o < nparts; o += kBT) {
      const PartRec pr = prow[o];
      if (pr.s != 0.0) t += pr.s * dexp2_call(((double)pr.m - (double)M) * rc.c_d);
    }
#pragma unroll 1
    for (int e = tid; e < nus; e += kBT) {
      const int l = s_ue[e].id - a.voff;
      const float zp = s_zp[e];
      // (binary32 MUFU exp2, like the stream's own terms: relative error ~2^-22 per term)
      if (l >= 0 && l < a.vloc && zp > -INFINITY) t += (double)ex2f((float)(((double)zp - (double)M) * rc.c_d));
    }
    for_long([&](int, int, float zp) {
      if (zp > -INFINITY) t += (double)ex2f((float)(((double)zp - (double)M) * rc.c_d));
    });
    return t;
  };
  const bool rowok = !bad && M > -INFINITY;
  uint32_t lo_k = kKey16NegInf + 1;
  float Tv = 0.f;
  bool take_all = false;
  uint64_t floor = 0;
  {
  // ---- bound: T = the K-th largest step key (each step key = the max of 1024 / 512 elements
  // rounded down, so K distinct elements are >= val(T)); every element >= val(T) lies in a
  // group with key >= T or is penalised.  One rank count per step key (smem broadcast).
  // Fallback (fewer than K finite step keys, or more steps than threads): T = the K-th largest
  // 16-bit key among the group keys and the penalised elements, by one histogram pass over the
  // kHistBins key steps below key(M) (one bin per key value: exact); a row whose K-th key lies
  // below that window takes every finite element (the collection then shrinks in bounded rounds).
  const uint32_t kmax = rowok ? key16_down(M) : 0u;
  bool need_hist = rowok;
  if (rowok && nsv >= keff && nsv <= kBT) {
    if (ctl[0] != 0) {
      lo_k = (uint32_t)ctl[0];
      need_hist = false;
    }
  }
  if (need_hist) {
    auto add_key = [&](uint32_t key) {
      const uint32_t d = kmax - key;
      if (key > kKey16NegInf && d < (uint32_t)kHistBins) atomicAdd(&hist[d], 1u);
    };
#pragma unroll 1
    for (int e = tid; e < nus; e += kBT) {
      const int l = s_ue[e].id - a.voff;
      const float zp = s_zp[e];
      if (l >= 0 && l < a.vloc && zp > -INFINITY && zp < INFINITY) add_key(key16_down(zp));
    }
    for_long([&](int, int, float zp) {
      if (zp > -INFINITY && zp < INFINITY) add_key(key16_down(zp));
    });
    for (int w = tid; w < gwords; w += kBT) {
      const uint4 g = (w < kSelGR * kBT) ? s_gk[w] : gk4[w];
      const uint32_t x[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        add_key(x[t] & 0xFFFFu);
        add_key(x[t] >> 16);
      }
    }
    cbar();
    // exclusive prefix over bins (bin 0 = key(M)): thread t owns bins [4t, 4t + 4)
    static_assert(kHistBins == 4 * kBT, "histogram scan layout");
    const uint4 hb = reinterpret_cast<const uint4*>(hist)[tid];
    const int own = (int)(hb.x + hb.y + hb.z + hb.w);
    const int incl = warp_incl_scan_i(own, lane);
    if (lane == 31) ms.bs.i[8 + (tid >> 5)] = incl;
    cbar();
    int before = incl - own;
    for (int w = 0; w < (tid >> 5); ++w) before += ms.bs.i[8 + w];
    if (tid == 0) ctl[0] = 0;
    cbar();
    if (before < keff && before + own >= keff) {
      const uint32_t h4[4] = {hb.x, hb.y, hb.z, hb.w};
      int cum = before, b = 0;
      while (cum + (int)h4[b] < keff) cum += (int)h4[b++];
      ctl[0] = (int)(kmax - (uint32_t)(4 * tid + b));
    }
    cbar();
    if (ctl[0] != 0) lo_k = (uint32_t)ctl[0];
  }
  // no bound (fewer than K finite keys, or the K-th below the histogram window): every finite
  // element is collected, so the candidate set is the complete row (a top-k row with
  // fewer than k finite logits is then decided here, not left pending)
  take_all = lo_k == kKey16NegInf + 1;
  Tv = take_all ? -FLT_MAX : key16_val(lo_k);
  // ---- collect: penalised elements (exact), then the qualifying groups (their re-read overlaps
  // the float64 softmax terms S = sum_parts s 2^((m - M) c) + sum_pen 2^((z' - M) c))
  auto push = [&](uint64_t c) {
    const int at = atomicAdd(&ctl[1], 1);
    if (at < kPool) ms.pool[at] = c;
  };
#pragma unroll 1
  for (int e = tid; e < nus; e += kBT) {
    const int l = s_ue[e].id - a.voff;
    if (l < 0 || l >= a.vloc) continue;
    const float zp = s_zp[e];
    if (zp >= Tv && zp > -INFINITY && zp < INFINITY) push(make_comp(zp, s_ue[e].id));
  }
  for_long([&](int id, int, float zp) {
    if (zp >= Tv && zp > -INFINITY && zp < INFINITY) push(make_comp(zp, id));
  });
  STR(19);
  const uint32_t lo2 = lo_k | (lo_k << 16);
  for (int base = 0; base < gwords; base += kSelGR * kBT) {
    uint4 gw[kSelGR];
#pragma unroll
    for (int q = 0; q < kSelGR; ++q) {
      const int w = base + tid + q * kBT;
      gw[q] = (base == 0) ? s_gk[tid + q * kBT] : (w < gwords) ? gk4[w] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < kSelGR; ++q) {
      const uint32_t w4[4] = {__vcmpgeu2(gw[q].x, lo2), __vcmpgeu2(gw[q].y, lo2), __vcmpgeu2(gw[q].z, lo2),
                              __vcmpgeu2(gw[q].w, lo2)};
      uint32_t bits = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) bits |= ((w4[t] & 1u) | ((w4[t] >> 30) & 2u)) << (2 * t);
      const int w = base + tid + q * kBT;
      const int cnt = __popc(bits);
      const int incl = warp_incl_scan_i(cnt, lane);
      const int tot = __shfl_sync(kFull, incl, 31);
      int at = 0;
      if (lane == 31 && tot) at = atomicAdd(&ctl[2], tot);
      at = __shfl_sync(kFull, at, 31) + incl - cnt;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        if (at < kSelQ) ql[at] = (uint32_t)(w * 8 + b);
        ++at;
      }
    }
  }
  cbar();
  STR(3);
  bool slow = ctl[2] > kSelQ;
  const int nq = slow ? 0 : ctl[2];
  for (int it0 = 0; it0 < nq * kG; it0 += kBT) {  // uniform per warp: aggregated pushes
    const int it = it0 + tid;
    const uint32_t g = (it < nq * kG) ? ql[it >> 2] : 0u;
    const int v = (int)(g >> 5) * kStepVec + (int)(g & 31) + 32 * (it & 3);
    const bool act = it < nq * kG && v < nvv;
    uint4 u4 = act ? ldg_stream(rowp + (int64_t)v * 16) : make_uint4(Dec<T>::kNegInfWord, Dec<T>::kNegInfWord,
                                                                       Dec<T>::kNegInfWord, Dec<T>::kNegInfWord);
    // the vector's penalised elements from the slot's presence bitmap (HistState::pmask), loaded
    // alongside the logits
    const int vk = v / kStepVec, vd = v - vk * kStepVec;
    const uint32_t pmw = act ? a.hs.pmask[((int64_t)slot * a.hs.spr + vk) * 32 + (vd & 31)] : 0u;
    if (it0 == 0) term = s_terms();  // the float64 softmax terms, while the re-read is in flight
    uint32_t msk = (pmw >> ((vd >> 5) * VEC)) & ((1u << VEC) - 1u);
#pragma unroll
    for (int t = 0; t < VEC; ++t)
      if (v * VEC + t >= a.vloc) msk |= 1u << t;
    if (msk) u4 = Dec<T>::mask(u4, msk);
    uint32_t sel = 0;
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      const float z = Dec<T>::elem(u4, t);
      if (act && z >= Tv && z > -INFINITY && z < INFINITY) sel |= 1u << t;
    }
    const int cnt = __popc(sel);
    const int incl = warp_incl_scan_i(cnt, lane);
    const int tot = __shfl_sync(kFull, incl, 31);
    int at = 0;
    if (lane == 31 && tot) at = atomicAdd(&ctl[1], tot);
    at = __shfl_sync(kFull, at, 31) + incl - cnt;
#pragma unroll
    for (int t = 0; t < VEC; ++t)
      if ((sel >> t) & 1u) {
        if (at < kPool) ms.pool[at] = make_comp(Dec<T>::elem(u4, t), a.voff + v * VEC + t);
        ++at;
      }
  }
  if (nq * kG == 0) term = s_terms();
  cbar();
  slow = slow || ctl[1] > kPool;  // uniform: after the barrier
  if (slow) floor = select_collect_slow<T>(a, rowp, utab, s_ue, nu, nus, prm, Tv, lo_k, nvv, gwords, keff, ms, ctl, ql);
  }
  const double S = block_sum_d(term, ms.bs);  // (its barriers also close the collection)
  // log S (only the decision's writer needs it): the last warp computes it while the others rank
  // the pool; read after the rank barrier
  if (tid >= kBT - 32) {
    const double l = dlog_call(S);
    if (tid == kBT - 1) *reinterpret_cast<double*>(ctl + 12) = l;
  }
  STR(4);
  // ---- exact top-K of the pool by rank counting
  // (each placed candidate's weight w = exp((z - M)/tau) in float64 is computed here, in
  // parallel, for the decision)
  const int nc = min(ctl[1], kPool);
  for (int i = tid; i < nc; i += kBT) {
    const uint64_t c = ms.pool[i];
    int rank = 0, j = 0;
    for (; j + 8 <= nc && rank < keff; j += 8) {
#pragma unroll
      for (int t = 0; t < 8; ++t) rank += ms.pool[j + t] > c ? 1 : 0;
    }
    for (; j < nc && rank < keff; ++j) rank += ms.pool[j] > c ? 1 : 0;
    if (rank < keff) {
      ms.top[rank] = c;
      // w = exp((z' - M)/tau) in float64 (R16: the kept-set weights, their top-p prefix
      // sums and the draw's CDF are float64-accurate, so a token may differ from the oracle's only
      // when a boundary lies within 1e-9 of it)
      ms.wv[rank] = rc.greedy ? 0.0 : dexp_call(((double)comp_val(c) - (double)M) / (double)rc.tau);
    }
  }
  cbar();
  STR(5);
  const int n = nc < keff ? nc : keff;
  // every element >= T is in the pool: the candidates are exact from the top down to T
  uint64_t F = (rowok && !take_all) ? make_comp(Tv, 0x7FFFFFFF) : 0ull;
  F = floor > F ? floor : F;
  if (nc > keff) F = ms.top[keff - 1] > F ? ms.top[keff - 1] : F;

  if (a.mode == 1) {  // ---- vocab-sharded phase 1: the row's candidate record
    RecHdr h;
    h.m = M;
    h.flags = bad ? kRecBad : 0u;
    h.s = S;
    h.R = __dmul_rn((double)M, rc.c_d);  // (rounded product: the merge subtracts the same rounded product)
    h.n = (uint32_t)n;
    h.rsv = 0;
    h.frontier = F;
    if (a.xp.world == 0) {
      uint8_t* out = a.out_records + (int64_t)r * a.out_stride;
      uint64_t* oe = reinterpret_cast<uint64_t*>(out + kRecHdrBytes);
      for (int i = tid; i < n; i += kBT) oe[i] = ms.top[i];
      if (tid == 0) *reinterpret_cast<RecHdr*>(out) = h;
      return;
    }
    // NEXT-2: the record goes straight into every peer's exchange buffer (P2P stores), then the
    // row's flag on every peer is raised (one system-scope release after the CTA barrier)
    const ExchPeers& x = a.xp;
    const uint32_t sq = x.seq[r] + 1;
    const int64_t off = (int64_t)(sq & 1) * x.par_pitch + (int64_t)x.rank * x.rank_pitch + (int64_t)r * x.row_stride;
    for (int p = 0; p < x.world; ++p) {
      uint8_t* out = x.bases[p] + off;
      uint64_t* oe = reinterpret_cast<uint64_t*>(out + kRecHdrBytes);
      for (int i = tid; i < n; i += kBT) oe[i] = ms.top[i];
      if (tid == 0) *reinterpret_cast<RecHdr*>(out) = h;
    }
    // every storing thread's own fence (a fence orders only its thread's writes), then the barrier,
    // then one release of the flags
    if (x.world > 1) __threadfence_system();
    else __threadfence();
    cbar();
    if (tid == 0) {  // release (system scope) after the CTA barrier: orders every thread's record stores
      x.seq[r] = sq;
      for (int p = 0; p < x.world; ++p)
        st_release_flag(reinterpret_cast<uint32_t*>(x.bases[p] + x.flags_off) + (int64_t)x.rank * x.nslots + r, sq,
                        x.world > 1);
    }
    if (!a.fuse_merge) return;
    // fused: every rank's record of this row (the peers' P2P stores land in this rank's buffer), then
    // the merge + decision + append of merge.cuh in this CTA (its shared memory is free again)
    if (tid == 0) {
      x.mseq[r] = sq;
      ctl[10] = exch_wait_row(x, r, sq);  // (ctl[10] is the decision's slot, unused in mode 1)
    }
    cbar();
    if (ctl[10]) {
      if (tid == 0) exch_timeout_row(a.ro, r);
      return;
    }
    const uint8_t* recs = x.bases[x.rank] + (int64_t)(sq & 1) * x.par_pitch + (int64_t)r * x.row_stride;
    block_merge_row(recs, x.rank_pitch, x.world, r, slot, prm, seed, a.step_dev ? *a.step_dev : a.step, a.V, a.kcand,
                    0, nullptr, a.ro, a.append, a.hs, false, invalid, ms, nullptr);
    return;
  }
  // ---- decision (whole block, candidate-parallel)
  STR(20);
  if (tid == 0) ctl[10] = -1;
  const double u = *reinterpret_cast<const double*>(ctl + 14);  // (warp kBW - 2, earlier)
  const double logS = *reinterpret_cast<const double*>(ctl + 12);
  STR(21);
  int32_t tok;
  {
    tok = block_decide(ms, ctl, n, M, S, logS, F, bad, invalid, rc, prm, u, r, a.ro, a.pending_ok != 0, tr);
  }
  STR(6);
  if (!a.append || tok < 0) return;
  if (nu > kSelPen) {
    block_append_global(a.hs, slot, tok);
    return;
  }
  block_append_smem(a.hs, slot, tok, smeta, s_ue, ms.bs);
  STR(7);
#undef STR
}

}  // namespace smp

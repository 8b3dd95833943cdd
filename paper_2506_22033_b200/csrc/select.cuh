// select.cuh — phase B of the sampling step: one CTA per row turns the row's piece records and
// group keys (phase A, stream.cuh) into the exact top-K candidates and the sample.
//
// One dependent chain per row, shaped for latency (the GPU is otherwise idle while it runs):
//   prologue   (independent of phase A; overlaps its tail under programmatic dependent launch)
//              the slot's unique-token table -> smem, raw logits of its ids -> registers
//   RT1        piece headers, lane-max lists, the row's group keys (one round trip)
//   bound      T = K-th largest lane max of the row (every list entry counts the entries >= it
//              across the lists by binary lifting).  K distinct elements are >= T.
//   collect    penalised ids: exact penalised value from the prefetched raws;
//              groups with key >= key(T): re-read (RT2), penalised ids and padding masked, every
//              element >= T pushed — the pool then holds EVERY element of the row >= T, exactly
//   top-K      rank counting over the pool (exact, ties impossible: composites are unique)
//   decide     warp 0 (merge.cuh warp_decide): top-k -> top-p -> min-p, Philox draw in id order
//   append     the sampled token into the slot's history (block-parallel shift from the smem copy)
// mode 1 (vocab-sharded phase 1) emits the row's candidate record instead of deciding.
#pragma once
#include "block.cuh"
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "philox.cuh"
#include "piece.cuh"

namespace smp {

constexpr int kSelPen = 2048;          // unique-token entries staged in smem
constexpr int kSelPR = kSelPen / kBT;  // raw penalised logits per thread (prefetch)
constexpr int kSelQ = 2048;            // qualifying-group list capacity
constexpr int kSelGR = 3;              // group-key words (8 keys) per thread per chunk

struct SelectArgs {
  const void* logits;
  int64_t ld;
  int B, V, voff, vloc;
  int64_t Vq, span, N;
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  int kcand, pen_mode, mode, append, pending_ok;
  HistState hs;
  const uint8_t* records;  // warp records (kWarpRecStride), index = global warp + row
  const uint16_t* gkeys;
  RowOut ro;
  uint8_t* out_records;  // mode 1: one candidate record per row
  int64_t out_stride;
  uint64_t* trace;       // debug: per-row phase timestamps (32 per row), nullable
};

// shared-memory carve-up (phase B)
constexpr int kSOffUe = 0;                                         // [kSelPen] UniqEntry
constexpr int kSOffLm = kSOffUe + kSelPen * 8;                     // [kMaxRecW][32] u32
constexpr int kSOffPool = kSOffLm + kMaxRecW * kLaneList * 4;      // [kPool] u64
constexpr int kSOffQl = kSOffPool + kPool * 8;                     // [kSelQ] u32
constexpr int kSOffTop = kSOffQl + kSelQ * 4;                      // [KC] u64
constexpr int kSOffWv = kSOffTop + SAMPLER_KCAND_MAX * 8;          // [KC] double
constexpr int kSOffById = kSOffWv + SAMPLER_KCAND_MAX * 8;         // [KC] u64
constexpr int kSOffHdr = kSOffById + SAMPLER_KCAND_MAX * 8;        // [kMaxRecW] RecHdr
constexpr int kSOffScr = kSOffHdr + kMaxRecW * 48;                 // f[8] d[8] u[16] i[16]
constexpr int kSOffCtl = kSOffScr + 288;                           // ints [16]
constexpr int kSOffGk = kSOffCtl + 64;                             // [kSelGR * kBT] uint4 group keys
constexpr int kSelectSmem = kSOffGk + kSelGR * kBT * 16;


// Append `tok` to the slot's history (P:371 incremental update) from the smem copy of the sorted
// unique-token table s_ue[0..nu) (nu <= kSelPen): one block-wide count, then every entry above the
// insertion point is stored one slot up straight from smem.
__device__ __forceinline__ void block_append_smem(const HistState& hs, int slot, int32_t tok, const SlotMeta& sm,
                                                  const UniqEntry* s_ue, const BlockScratch& bs) {
  const int tid = threadIdx.x;
  const int nu = sm.n_uniq, np = sm.n_prompt, no = sm.n_out;
  if (np + no + 1 > hs.L) {
    if (tid == 0) hs.meta[slot].flags |= 1;
    return;
  }
  int cl = 0;
  for (int i = tid; i < nu; i += kBT) cl += (s_ue[i].id < tok ? 1 : 0) + (s_ue[i].id == tok ? (1 << 20) : 0);
  const int cs = block_sum_i(cl, bs);
  const int less = cs & ((1 << 20) - 1);
  const bool found = (cs >> 20) != 0;
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
  const uint16_t* gk = a.gkeys + (int64_t)blockIdx.x * (a.Vq / kG);
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

template <typename T>
__global__ void __launch_bounds__(kBT, 2) select_rows_kernel(const SelectArgs a) {
  constexpr int VEC = Dec<T>::N;
  constexpr int ESZ = (int)sizeof(T);
  extern __shared__ __align__(128) uint8_t smem[];
  const int r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  UniqEntry* s_ue = reinterpret_cast<UniqEntry*>(smem + kSOffUe);
  uint32_t* lm = reinterpret_cast<uint32_t*>(smem + kSOffLm);
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

  // ---- prologue: nothing here depends on phase A
  const int slot = a.slots ? a.slots[r] : r;
  const sampling_params prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
  const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
  const RowCfg rc = decode_row(prm, a.V, a.kcand);
  const int keff = rc.keff;
  const SlotMeta smeta = a.hs.meta[slot];
  const int nu = smeta.n_uniq;
  const int nus = min(nu, kSelPen);
  const UniqEntry* utab = a.hs.uniq + (int64_t)slot * a.hs.L;
  const uint8_t* rowp = reinterpret_cast<const uint8_t*>(a.logits) + (int64_t)r * a.ld * ESZ;
  float raw[kSelPR];
  int lid[kSelPR];
#pragma unroll
  for (int q = 0; q < kSelPR; ++q) {
    const int e = tid + q * kBT;
    lid[q] = -1;
    raw[q] = 0.f;
    if (e < nus) {
      const UniqEntry ue = utab[e];
      s_ue[e] = ue;
      const int l = ue.id - a.voff;
      if (l >= 0 && l < a.vloc) {
        lid[q] = l;
        raw[q] = Dec<T>::load1(rowp, l);
      }
    }
  }
  if (tid == 0) {
    ctl[0] = 0;
    ctl[1] = 0;
    ctl[2] = 0;
    ctl[5] = 0;
  }
  griddep_wait();  // phase A's records and group keys are visible from here on
  // ---- RT1: warp-record headers, lane-max lists, group keys
  const int64_t w_first = ((int64_t)r * a.Vq) / a.span;
  const int64_t w_last = ((int64_t)(r + 1) * a.Vq - 1) / a.span;
  const int nrec = (int)(w_last - w_first + 1);  // <= kMaxRecW (plan)
  const uint8_t* recs = a.records + (w_first + r) * (int64_t)kWarpRecStride;
  if (tid < nrec) ms.hdr[tid] = *reinterpret_cast<const RecHdr*>(recs + (int64_t)tid * kWarpRecStride);
  for (int i = tid; i < nrec * kLaneList; i += kBT)
    lm[i] = reinterpret_cast<const uint32_t*>(recs + (int64_t)(i >> 5) * kWarpRecStride + kRecHdrBytes)[i & 31];
  const int nvv = (a.vloc + VEC - 1) / VEC;
  const int gwords = ((nvv + kStepVec - 1) / kStepVec) * 32 / 8;  // valid group-key words (8 keys)
  const uint4* gk4 = reinterpret_cast<const uint4*>(a.gkeys + (int64_t)r * (a.Vq / kG));
  uint4* s_gk = reinterpret_cast<uint4*>(smem + kSOffGk);
#pragma unroll
  for (int q = 0; q < kSelGR; ++q) {  // staged in smem: every load of RT1 completes at one barrier
    const int w = tid + q * kBT;
    s_gk[w] = (w < gwords) ? gk4[w] : make_uint4(0, 0, 0, 0);
  }
  cbar();
  STR(1);
  // ---- bound: T = K-th largest lane max of the row; M, S, flags (warp 0)
  // prefilter (every thread, smem broadcast): with m = ceil(K / nrec), the lists holding >= m
  // entries contribute m entries each >= LB = min of their m-th entries; if that is >= K
  // entries, T >= LB and only entries >= LB need an exact count
  uint32_t lb = 0;
  {
    const int m = (keff + nrec - 1) / nrec;
    uint32_t mn = 0xFFFFFFFFu;
    int have = 0;
    if (m <= kLaneList)
      for (int o = 0; o < nrec; ++o)
        if ((int)ms.hdr[o].n >= m) {
          mn = min(mn, lm[o * kLaneList + m - 1]);
          have += m;
        }
    if (have >= keff) lb = mn;
  }
  // the entries >= LB, compacted (warp-aggregated), then one exact count per entry
  uint32_t* cx = ql;  // scratch until the collect phase
  for (int i0 = 0; i0 < nrec * kLaneList; i0 += kBT) {
    const int i = i0 + tid;
    const uint32_t x = (i < nrec * kLaneList) ? lm[i] : 0u;
    const bool pass = x != 0u && x >= lb;
    const unsigned bal = __ballot_sync(kFull, pass);
    int at = 0;
    if (lane == 0 && bal) at = atomicAdd(&ctl[5], __popc(bal));
    at = __shfl_sync(kFull, at, 0) + __popc(bal & ((1u << lane) - 1u));
    if (pass) cx[at] = x;
  }
  cbar();
  const int ncx = ctl[5];
  uint32_t tbest = 0;  // largest own entry with count >= K (warp-reduced: one atomic per warp)
  for (int j = tid; j < ncx; j += kBT) {
    const uint32_t x = cx[j];
    if (x <= tbest) continue;
    int c = 0;
    for (int o0 = 0; o0 < nrec; o0 += 8) {  // 8 lists side by side (independent lifting chains)
      int pos[8], no[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        pos[t] = 0;
        no[t] = (o0 + t < nrec) ? (int)ms.hdr[o0 + t].n : 0;
      }
#pragma unroll
      for (int st = 32; st; st >>= 1)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (pos[t] + st <= no[t] && lm[(o0 + t) * kLaneList + pos[t] + st - 1] >= x) pos[t] += st;
#pragma unroll
      for (int t = 0; t < 8; ++t) c += pos[t];
    }
    if (c >= keff) tbest = x;
  }
  STR(16);
  tbest = __reduce_max_sync(kFull, tbest);
  if (lane == 0 && tbest) atomicMax(reinterpret_cast<unsigned*>(&ctl[0]), tbest);
  STR(17);
  if (tid >= kBT - 32) {  // the last warp (the counting above uses the first warps)
    float mloc = -INFINITY;
    unsigned fl = 0;
    for (int o = lane; o < nrec; o += 32) {
      mloc = fmaxf(mloc, ms.hdr[o].m);
      fl |= ms.hdr[o].flags;
    }
    const float M = warp_max(mloc);
    const double RM = (double)M * rc.c_d;
    double term = 0.0;
    for (int o = lane; o < nrec; o += 32)
      if (ms.hdr[o].s != 0.0) term += ms.hdr[o].s * exp2(ms.hdr[o].R - RM);
    const double S = warp_sum_d(term);
    fl = __reduce_or_sync(kFull, fl);
    if (lane == 0) {
      ms.bs.f[0] = M;
      ms.bs.d[0] = S;
      ms.bs.d[1] = log(S);
      ms.bs.i[0] = (int)fl;
    }
    STR(18);
  }
  cbar();
  STR(2);
  const float M = ms.bs.f[0];  // (the block scratch is reused below)
  const double S = ms.bs.d[0];
  const double logS = ms.bs.d[1];
  const bool bad = (ms.bs.i[0] & kRecBad) != 0;
  const uint32_t tkey = (uint32_t)ctl[0];
  const bool bounded = tkey != 0u;
  const float Tv = bounded ? key2f(tkey) : -3.402823466e38f;
  const uint32_t lo_k = bounded ? max(key16_down(Tv), kKey16NegInf + 1) : kKey16NegInf + 1;
  // ---- collect: penalised elements (exact), then the qualifying groups
  auto push = [&](uint64_t c) {
    const int at = atomicAdd(&ctl[1], 1);
    if (at < kPool) ms.pool[at] = c;
  };
#pragma unroll
  for (int q = 0; q < kSelPR; ++q) {
    if (lid[q] < 0) continue;
    const float zp = apply_penalty(raw[q], s_ue[tid + q * kBT].meta, prm, a.pen_mode);
    if (zp >= Tv && zp > -INFINITY && zp < INFINITY) push(make_comp(zp, a.voff + lid[q]));
  }
  for (int e = kSelPen + tid; e < nu; e += kBT) {  // very long tables: straight from global
    const UniqEntry ue = utab[e];
    const int l = ue.id - a.voff;
    if (l < 0 || l >= a.vloc) continue;
    const float zp = apply_penalty(Dec<T>::load1(rowp, l), ue.meta, prm, a.pen_mode);
    if (zp >= Tv && zp > -INFINITY && zp < INFINITY) push(make_comp(zp, ue.id));
  }
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
  const bool slow = ctl[2] > kSelQ || ctl[1] + ctl[2] * kG * VEC > kPool;
  const int nq = slow ? 0 : ctl[2];
  const int ns = nus;
  for (int it0 = 0; it0 < nq * kG; it0 += kBT) {  // uniform per warp: aggregated pushes
    const int it = it0 + tid;
    const uint32_t g = (it < nq * kG) ? ql[it >> 2] : 0u;
    const int v = (int)(g >> 5) * kStepVec + (int)(g & 31) + 32 * (it & 3);
    const bool act = it < nq * kG && v < nvv;
    uint4 u4 = act ? ldg_stream(rowp + (int64_t)v * 16) : make_uint4(Dec<T>::kNegInfWord, Dec<T>::kNegInfWord,
                                                                       Dec<T>::kNegInfWord, Dec<T>::kNegInfWord);
    uint32_t msk = listed_mask<VEC>(s_ue, ns, a.voff + v * VEC);
#pragma unroll
    for (int t = 0; t < VEC; ++t)
      if (v * VEC + t >= a.vloc) msk |= 1u << t;
    if (nu > kSelPen)  // very long tables: the tail entries are in global memory only
      for (int e = kSelPen; e < nu; ++e) {
        const int k = utab[e].id - a.voff - v * VEC;
        if (k >= 0 && k < VEC) msk |= 1u << k;
      }
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
  uint64_t floor = 0;
  if (slow) floor = select_collect_slow<T>(a, rowp, utab, s_ue, nu, nus, prm, Tv, lo_k, nvv, gwords, keff, ms, ctl, ql);
  cbar();
  STR(4);
  // ---- exact top-K of the pool by rank counting
  // (each placed candidate's weight w = exp((z - M)/tau) in float64 is computed here, in
  // parallel, for the decision)
  const int nc = min(ctl[1], kPool);
  const double inv_tau = 1.0 / (double)rc.tau;
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
      ms.wv[rank] = rc.greedy ? 0.0 : exp(((double)comp_val(c) - (double)M) * inv_tau);
    }
  }
  cbar();
  STR(5);
  const int n = nc < keff ? nc : keff;
  // every element >= T is in the pool: the candidates are exact from the top down to T
  uint64_t F = bounded ? make_comp(Tv, 0x7FFFFFFF) : 0ull;
  F = floor > F ? floor : F;
  if (nc > keff) F = ms.top[keff - 1] > F ? ms.top[keff - 1] : F;

  if (a.mode == 1) {  // ---- vocab-sharded phase 1: the row's candidate record
    uint8_t* out = a.out_records + (int64_t)r * a.out_stride;
    uint64_t* oe = reinterpret_cast<uint64_t*>(out + kRecHdrBytes);
    for (int i = tid; i < n; i += kBT) oe[i] = ms.top[i];
    if (tid == 0) {
      RecHdr h;
      h.m = M;
      h.flags = bad ? kRecBad : 0u;
      h.s = S;
      h.R = (double)M * rc.c_d;
      h.n = (uint32_t)n;
      h.rsv = 0;
      h.frontier = F;
      *reinterpret_cast<RecHdr*>(out) = h;
    }
    return;
  }
  // ---- decision (warp 0)
  if (tid < 32) {
    const double u = philox_uniform(seed, prm.request_id, a.step);
    const int t = warp_decide(ms, n, M, S, F, bad, rc, prm, seed, a.step, r, a.ro, a.pending_ok != 0, tr, true,
                              logS, u);
    if (lane == 0) ctl[3] = t;
  }
  STR(6);
  cbar();
  const int32_t tok = ctl[3];
  if (!a.append || tok < 0) return;
  if (nu > kSelPen) {
    if (tid < 32) warp_append_token(a.hs, slot, tok, lane);
    return;
  }
  block_append_smem(a.hs, slot, tok, smeta, s_ue, ms.bs);
  STR(7);
#undef STR
}

}  // namespace smp

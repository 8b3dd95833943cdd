// stream.cuh — phase A of the sampling step: one streaming pass over the logits [B x V].
//
// Every warp works alone (piece.cuh: the padded [B x Vq] vector space cut into equal STEP-
// aligned warp spans; a span crossing a row boundary yields one sub-piece per row) — there is no
// CTA barrier in phase A, so no warp ever waits for another's epilogue or metadata:
//   * metadata: the row's params and the slot's incremental unique-token table: the
//     warp counts the entries below / inside its sub-piece and stages those into its own smem
//     region; the raw logits of the penalised ids are prefetched into registers.
//   * the stream: 16-byte read-only no-L1-allocate loads, 4 vectors (32 bf16 / 16 f32 logits)
//     per lane per step, the next step's loads issued before the current step is computed; the
//     penalised ids and the padding tail are masked to -inf in registers (the staged ids walked
//     in order with the stream), then one NaN-propagating max per vector, the group key (bf16
//     key of the group max, rounded down) stored to gkeys[row], and the exp-sum: 2 FFMA + 1
//     MUFU.EX2 per logit into a float64 lane accumulator with an integer exponent reference.
//   * the penalised elements enter as single exact values: OPENAI_CTRL / LINEAR penalty in
//     exact binary32 ops, exp-sum, lane max.
//   * epilogue: the 32 lane maxima sorted by a shuffle bitonic network and written with the
//     sub-piece's max / exp-sum / bad flag as the warp record.
// The selection (bound, re-read of the qualifying groups, exact top-K, decision, draw) is phase B
// (select.cuh).
#pragma once
#include "common.cuh"
#include "elem.cuh"
#include "merge.cuh"
#include "piece.cuh"

namespace smp {

constexpr int kWarpsPerCta = 8;
constexpr int kCtasPerSm = 3;
constexpr int kPenW = 128;         // penalty entries staged per warp (more: read from global)
constexpr int kPenWQ = kPenW / 32;  // raw penalised logits prefetched per lane
constexpr int kStreamSmem = kWarpsPerCta * kPenW * 8;

struct StreamArgs {
  const void* logits;
  int64_t ld;          // row stride (elements)
  int B;
  int V;               // global vocab
  int voff, vloc;      // local slice
  int64_t Vq;          // padded row length in vectors (multiple of kStepVec)
  int64_t span;        // vectors per warp (multiple of kStepVec)
  int64_t N;           // B * Vq
  const int32_t* slots;
  const sampling_params* params_dev;  // nullable
  const sampling_params* params_tab;
  int kcand;
  int pen_mode;
  HistState hs;
  uint8_t* records;    // warp records (kWarpRecStride bytes), index = global warp + row
  uint16_t* gkeys;     // [B][Vq / 4] group keys
  uint64_t* trace;     // debug: per-warp start / end timestamps (globaltimer ns, 8 per warp), nullable
};

template <typename T>
__global__ void __launch_bounds__(kWarpsPerCta * 32, kCtasPerSm) stream_kernel(const StreamArgs a) {
  constexpr int VEC = Dec<T>::N;
  constexpr int ESZ = (int)sizeof(T);

  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + wid;  // global warp index
  const uint4 kNegInfVec = make_uint4(Dec<T>::kNegInfWord, Dec<T>::kNegInfWord, Dec<T>::kNegInfWord,
                                      Dec<T>::kNegInfWord);
  griddep_launch();  // phase B's CTAs may be scheduled as this grid's CTAs retire
  const int64_t a0 = gw * a.span;
  const int64_t a1 = min(a.N, a0 + a.span);
  UniqEntry* wpen = reinterpret_cast<UniqEntry*>(smem) + wid * kPenW;
  const uint8_t* lg = reinterpret_cast<const uint8_t*>(a.logits);
  const int nvv = (a.vloc + VEC - 1) / VEC;  // real vectors per row
  if (a.trace && lane == 0) a.trace[gw * 8 + 0] = gtimer();

  int64_t pos = a0;
  while (pos < a1) {
    // ---------------- sub-piece = row vectors [p0, p1) of row r (STEP-aligned)
    const int r = (int)(pos / a.Vq);
    const int p0 = (int)(pos - (int64_t)r * a.Vq);
    const int64_t pend = min(a1, (int64_t)(r + 1) * a.Vq);
    const int p1 = (int)(pend - (int64_t)r * a.Vq);
    const int pv1 = min(p1, nvv);  // real vectors end
    const int nsteps = pv1 > p0 ? (pv1 - p0 + kStepVec - 1) / kStepVec : 0;
    const uint8_t* rowp = lg + (int64_t)r * a.ld * ESZ;
    // first loads go out before any metadata round trip
    uint4 u[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int v = p0 + lane + 32 * j;
      u[j] = (nsteps > 0 && v < nvv) ? ldg_stream(rowp + (int64_t)v * 16) : kNegInfVec;
    }
    const int slot = a.slots ? a.slots[r] : r;
    const sampling_params* gprm = a.params_dev ? a.params_dev + r : a.params_tab + slot;
    const RowCfg rc = decode_row(*gprm, a.V, a.kcand);
    // penalty entries of the sub-piece: global ids in [g0, g1)
    const UniqEntry* utab = a.hs.uniq + (int64_t)slot * a.hs.L;
    const int nu = a.hs.meta[slot].n_uniq;
    const int g0 = a.voff + p0 * VEC, g1 = a.voff + min(pv1 * VEC, a.vloc);
    int lo = 0, hi = 0;
    for (int i = lane; i < nu; i += 32) {
      const int id = utab[i].id;
      lo += id < g0;
      hi += id < g1;
    }
    lo = warp_sum_i(lo);
    hi = warp_sum_i(hi);
    const int pcount = max(0, hi - lo);
    const bool staged = pcount <= kPenW;
    const UniqEntry* psrc = staged ? wpen : utab + lo;
    if (staged)
      for (int i = lane; i < pcount; i += 32) wpen[i] = utab[lo + i];
    __syncwarp();
    // raw logits of the penalised ids (scattered single elements): issued now, consumed after
    // the stream, so their latency hides under it
    float praw[kPenWQ];
#pragma unroll
    for (int q = 0; q < kPenWQ; ++q) {
      const int e = lane + 32 * q;
      praw[q] = (e < pcount) ? Dec<T>::load1(rowp, psrc[e].id - a.voff) : 0.f;
    }
    LaneAcc la;
    la.reset();
    int wcur = 0;
    int next_pen = (pcount > 0) ? psrc[0].id - a.voff : 0x7FFFFFFF;  // row-local element id
    uint16_t* gk = a.gkeys + (int64_t)r * (a.Vq / kG);

    // ================= the stream =================
    for (int k = 0; k < nsteps; ++k) {
      const int vb = p0 + k * kStepVec;      // row vector index of the step
      const int s1 = (vb + kStepVec) * VEC;  // row-local element end of the step
      uint4 cur[kG];  // this step's vectors (past the row: -inf)
#pragma unroll
      for (int j = 0; j < kG; ++j) cur[j] = u[j];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int v = vb + kStepVec + lane + 32 * j;
        u[j] = (k + 1 < nsteps && v < nvv) ? ldg_stream(rowp + (int64_t)v * 16) : kNegInfVec;
      }
      // penalised ids and the padding tail are masked to -inf here (bit j*VEC+t of pm); the
      // penalised elements enter the sums and the candidates as single exact values instead
      uint32_t pm = 0;
      while (next_pen < s1) {
        const int d = next_pen / VEC - vb;  // vector offset within the step
        if ((d & 31) == lane) pm |= 1u << ((d >> 5) * VEC + (next_pen & (VEC - 1)));
        ++wcur;
        next_pen = (wcur < pcount) ? psrc[wcur].id - a.voff : 0x7FFFFFFF;
      }
      if (s1 > a.vloc) {
#pragma unroll
        for (int j = 0; j < kG; ++j)
#pragma unroll
          for (int t = 0; t < VEC; ++t)
            if ((vb + lane + 32 * j) * VEC + t >= a.vloc) pm |= 1u << (j * VEC + t);
      }
      if (pm) {
#pragma unroll
        for (int j = 0; j < kG; ++j) {
          const uint32_t b = (pm >> (j * VEC)) & ((1u << VEC) - 1u);
          if (b) cur[j] = Dec<T>::mask(cur[j], b);
        }
      }
      float vm[kG];
#pragma unroll
      for (int j = 0; j < kG; ++j) vm[j] = Dec<T>::vmax(cur[j]);
      const float gm = fmax_nan(fmax_nan(vm[0], vm[1]), fmax_nan(vm[2], vm[3]));
      la.bad |= !(gm < INFINITY) ? 1 : 0;  // NaN or +inf in the group
      gk[vb / kG + lane] = (uint16_t)key16_down(gm);
      const float gmax = fmaxf(fmaxf(vm[0], vm[1]), fmaxf(vm[2], vm[3]));
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
    // penalised elements: exact values (OPENAI_CTRL / LINEAR) into the lane sums
    // and maxima
    if (pcount > 0) {
      const sampling_params prm = *gprm;
      for (int q = 0; lane + 32 * q < pcount; ++q) {
        const int e = lane + 32 * q;
        const UniqEntry ue = psrc[e];
        float raw = 0.f;
#pragma unroll
        for (int qq = 0; qq < kPenWQ; ++qq)
          if (qq == q) raw = praw[qq];
        if (q >= kPenWQ) raw = Dec<T>::load1(rowp, ue.id - a.voff);
        la.bad |= !(raw < INFINITY) ? 1 : 0;
        const float zp = apply_penalty(raw, ue.meta, prm, a.pen_mode);
        la.bad |= !(zp < INFINITY) ? 1 : 0;
        if (zp > -INFINITY && zp < INFINITY) {
          if (zp > la.thr) lane_rebase(la, zp, rc);
          la.acc += (double)lane_exp(zp, la, rc);
          la.mmax = fmaxf(la.mmax, zp);
        }
      }
    }
    // ================= epilogue: the warp record =================
    uint32_t x = (la.mmax > -INFINITY) ? f2key(la.mmax) : 0u;  // 0 = no finite element
    x = warp_sort_desc_u32(x, lane);
    const float m = warp_max(la.mmax);
    const float Rl = warp_max(la.acc != 0.0 ? la.R : -INFINITY);
    double sv = (la.acc != 0.0) ? scale_pow2(la.acc, la.R - Rl) : 0.0;
    sv = warp_sum_d(sv);
    const int bad = __any_sync(kFull, la.bad);
    const int cnt = __popc(__ballot_sync(kFull, x != 0u));
    uint8_t* rec = a.records + (gw + r) * (int64_t)kWarpRecStride;
    reinterpret_cast<uint32_t*>(rec + kRecHdrBytes)[lane] = x;
    if (lane == 0) {
      RecHdr h;
      h.m = m;
      h.flags = bad ? kRecBad : 0u;
      h.s = sv;
      h.R = (double)Rl;
      h.n = (uint32_t)cnt;
      h.rsv = 0;
      h.frontier = 0;
      *reinterpret_cast<RecHdr*>(rec) = h;
    }
    __syncwarp();  // the staged entries are rewritten by the next sub-piece
    pos = pend;
  }
  if (a.trace && lane == 0) a.trace[gw * 8 + 7] = gtimer();
}

}  // namespace smp

// merge.cuh — per-row merge of partial records and the final filter + draw (one CTA per row).
//
// A row's partial records (CTA pieces of one GPU's stream, or one record per vocab shard after
// the all-gather) each carry (m, R, s, top-K candidates sorted descending, frontier).
// The merge combines, in fixed record order (deterministic),
//     M = max m_i,   S = sum_i s_i * 2^(R_i - M*log2(e)/tau)           (float64)
// and the union of candidates by rank-merging the sorted lists (every element's rank = its
// position in its own list + a binary search in each other list), exact down to the max
// frontier; then — in the order of DESIGN.md R6 — top-k -> top-p (renormalised over the
// top-k survivors, R7/R8) -> min-p, and an inverse-CDF draw over the kept set in ascending
// id order with a Philox uniform (R10, R11).  Candidate weights
// w_i = exp((z'_i - M)/tau) are float64.
#pragma once
#include "block.cuh"
#include "common.cuh"
#include "philox.cuh"

namespace smp {

constexpr int kMaxRec = 16;    // records merged per row (pieces per row / shards)
constexpr int kPool = 2048;    // candidate union capacity

struct RowOut {
  int32_t* tokens;
  float* logprobs;
  float* flogprobs;  // nullable
  int32_t* status;   // nullable
  RowInfo* info;     // per-row hand-off / debug
};

struct HistState {
  SlotMeta* meta;
  UniqEntry* uniq;
  int32_t* tokens;
  int L;
};

struct MergeSmem {
  uint64_t* pool;   // [kPool]
  uint64_t* top;    // [SAMPLER_KCAND_MAX]
  double* wv;       // [SAMPLER_KCAND_MAX]
  uint64_t* byid;   // [SAMPLER_KCAND_MAX]
  RecHdr* hdr;      // [kMaxRec]
  int* off;         // [kMaxRec + 1]
  BlockScratch bs;
};
constexpr int kMergeSmemBytes = kPool * 8 + 3 * SAMPLER_KCAND_MAX * 8 + kMaxRec * 48 + (kMaxRec + 1) * 4 + 12;

// Incremental penalty-table update for one appended token ("only the B elements of f
// that correspond to the newly generated token IDs are incrementally updated").  One warp.
__device__ __forceinline__ void warp_append_token(const HistState& hs, int slot, int32_t tok, int lane) {
  SlotMeta* sm = hs.meta + slot;
  const int np = sm->n_prompt, no = sm->n_out, nu = sm->n_uniq;
  if (np + no + 1 > hs.L) {
    if (lane == 0) sm->flags |= 1;
    return;
  }
  UniqEntry* u = hs.uniq + (int64_t)slot * hs.L;
  int less = 0;
  for (int i = lane; i < nu; i += 32) less += (u[i].id < tok) ? 1 : 0;
  less = warp_sum_i(less);
  const bool found = (less < nu) && (u[less].id == tok);
  __syncwarp();
  if (found) {
    if (lane == 0) u[less].meta += 2u;
  } else {
    for (int top = nu; top > less; top -= 32) {
      const int i = top - 1 - lane;
      UniqEntry e;
      const bool act = i >= less;
      if (act) e = u[i];
      __syncwarp();
      if (act) u[i + 1] = e;
      __syncwarp();
    }
    if (lane == 0) {
      UniqEntry e;
      e.id = tok;
      e.meta = 2u;
      u[less] = e;
    }
  }
  if (lane == 0) {
    hs.tokens[(int64_t)slot * hs.L + np + no] = tok;
    sm->n_out = no + 1;
    if (!found) sm->n_uniq = nu + 1;
  }
  __syncwarp();
}

// number of entries of the descending list L[0..n) strictly greater than c
__device__ __forceinline__ int count_gt(const uint64_t* L, int n, uint64_t c) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (L[mid] > c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge `nrec` records (pitch `pitch` bytes, first at `recs`) of one row; all kBT threads.
// mode 0: final decision + outputs (+ append).  mode 1: write one merged record to out_rec.
__device__ __noinline__ void block_merge_row(const uint8_t* recs, int64_t pitch, int nrec, int row, int slot,
                                             const sampling_params& p, uint64_t seed, uint64_t step, int V,
                                             int kcand, int mode, uint8_t* out_rec, const RowOut& ro, int append,
                                             const HistState& hs, bool pending_ok, const MergeSmem& ms) {
  const RowCfg rc = decode_row(p, V, kcand);
  const int tid = threadIdx.x, lane = tid & 31;
  const int keff = rc.keff;
  // ---- headers
  if (tid < nrec) ms.hdr[tid] = *reinterpret_cast<const RecHdr*>(recs + (int64_t)tid * pitch);
  cbar();
  if (tid == 0) {
    int o = 0;
    for (int i = 0; i < nrec; ++i) {
      ms.off[i] = o;
      const int n = (int)ms.hdr[i].n < keff ? (int)ms.hdr[i].n : keff;
      o += n;
    }
    ms.off[nrec] = o;
  }
  cbar();
  const int U = ms.off[nrec];
  // ---- load the (sorted) lists into the pool
  for (int i = 0; i < nrec; ++i) {
    const uint64_t* e = rec_entries(recs + (int64_t)i * pitch);
    const int o = ms.off[i], n = ms.off[i + 1] - o;
    for (int j = tid; j < n; j += kBT) ms.pool[o + j] = e[j];
  }
  cbar();
  // ---- rank-merge: element at position q of list i has rank q + sum_{j != i} count_gt(list j)
  for (int i = 0; i < nrec; ++i) {
    const int o = ms.off[i], n = ms.off[i + 1] - o;
    for (int q = tid; q < n; q += kBT) {
      const uint64_t c = ms.pool[o + q];
      int rank = q;
      for (int j = 0; j < nrec && rank < keff; ++j)
        if (j != i) rank += count_gt(ms.pool + ms.off[j], ms.off[j + 1] - ms.off[j], c);
      if (rank < keff) ms.top[rank] = c;
    }
  }
  cbar();
  const int n = U < keff ? U : keff;
  // ---- M, S, frontier (fixed record order)
  if (tid == 0) {
    float M = -INFINITY;
    uint32_t fl = 0;
    uint64_t F = 0;
    for (int i = 0; i < nrec; ++i) {
      M = fmaxf(M, ms.hdr[i].m);
      fl |= ms.hdr[i].flags;
      F = ms.hdr[i].frontier > F ? ms.hdr[i].frontier : F;
    }
    const double RM = (double)M * rc.c_d;
    double S = 0.0;
    for (int i = 0; i < nrec; ++i)
      if (ms.hdr[i].s != 0.0) S += ms.hdr[i].s * exp2(ms.hdr[i].R - RM);
    if (U > keff && n > 0) F = ms.top[n - 1] > F ? ms.top[n - 1] : F;
    ms.bs.f[0] = M;
    ms.bs.d[0] = S;
    ms.bs.u[0] = F;
    ms.bs.i[0] = (int)fl;
  }
  cbar();
  const float M = ms.bs.f[0];
  const double S = ms.bs.d[0];
  const uint64_t F = ms.bs.u[0];
  const bool bad = (ms.bs.i[0] & kRecBad) != 0;
  cbar();

  if (mode == 1) {  // ---- local merge: emit one record
    uint64_t* oe = reinterpret_cast<uint64_t*>(out_rec + kRecHdrBytes);
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
      *reinterpret_cast<RecHdr*>(out_rec) = h;
    }
    cbar();
    return;
  }

  // ---- final decision (warp 0; the other warps compute weights first)
  const double inv_tau = 1.0 / (double)rc.tau;
  for (int i = tid; i < n; i += kBT) ms.wv[i] = exp(((double)comp_val(ms.top[i]) - (double)M) * inv_tau);
  cbar();
  if (tid < 32) {
    int status = SAMPLER_ROW_OK;
    if (bad)
      status = SAMPLER_ROW_NONFINITE;
    else if (n == 0 || !(M > -INFINITY))
      status = SAMPLER_ROW_ALL_NEG_INF;
    int32_t tok = -1;
    double lp = NAN, flp = NAN, W = 0.0;
    uint64_t cutoff = 0;
    if (status == SAMPLER_ROW_OK) {
      int n_exact = 0;
      for (int i = lane; i < n; i += 32) n_exact += (ms.top[i] >= F) ? 1 : 0;
      n_exact = warp_sum_i(n_exact);
      const bool complete = (F == 0);
      int n3 = -1;
      if (rc.greedy) {
        n3 = 1;
      } else {
        const int UNK = 0x7FFFFFFF;
        int n1 = UNK;
        if (rc.topk_on) {
          if (rc.k <= n_exact) n1 = rc.k;
          else if (complete) n1 = n;
        } else if (complete) {
          n1 = n;
        }
        int cand = n1;
        bool ok = true;
        if (rc.top_p < 1.0f) {
          double W1 = 0.0;
          bool w1k = false;
          if (n1 != UNK) {
            double a = 0.0;
            for (int i = lane; i < n1; i += 32) a += ms.wv[i];
            W1 = warp_sum_d(a);
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
            int n2 = UNK;
            double run = 0.0;
            for (int base = 0; base < lim && n2 == UNK; base += 32) {
              const int i = base + lane;
              const double x = (i < lim) ? ms.wv[i] : 0.0;
              const double c = run + warp_incl_scan_d(x, lane);
              const unsigned hit = __ballot_sync(kFull, (i < lim) && (c >= target));
              if (hit) n2 = base + __ffs(hit);
              run = __shfl_sync(kFull, c, 31);
            }
            if (n2 == UNK && n1 != UNK && n1 <= n_exact) n2 = n1;  // rounding shortfall
            if (n2 != UNK) cand = cand < n2 ? cand : n2;
          }
        }
        if (ok && rc.min_p > 0.0f) {
          int nm = UNK;
          for (int base = 0; base < n_exact && nm == UNK; base += 32) {
            const int i = base + lane;
            const unsigned hit = __ballot_sync(kFull, (i < n_exact) && (ms.wv[i] < (double)rc.min_p));
            if (hit) nm = base + __ffs(hit) - 1;
          }
          if (nm == UNK && complete) nm = n;
          if (nm != UNK) cand = cand < nm ? cand : nm;
        }
        if (ok && cand != UNK && cand <= n_exact && cand >= 1) n3 = cand;
      }
      if (n3 < 0) {
        status = kRowPending;
      } else {
        cutoff = ms.top[n3 - 1];
        if (rc.greedy) {
          tok = comp_id(ms.top[0]);
          W = 1.0;
          lp = ((double)comp_val(ms.top[0]) - (double)M) - log(S);
          flp = 0.0;
        } else {
          // kept set K3 = first n3 of pi, walked in ascending id order (R10); rank by id
          for (int i = lane; i < n3; i += 32)
            ms.byid[i] = ((uint64_t)(uint32_t)comp_id(ms.top[i]) << 32) | (uint32_t)i;
          __syncwarp();
          int N = 1;
          while (N < n3) N <<= 1;
          for (int i = n3 + lane; i < N; i += 32) ms.byid[i] = ~0ull;
          __syncwarp();
          for (int k = 2; k <= N; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
              for (int i = lane; i < N; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                  const uint64_t a = ms.byid[i], b = ms.byid[ixj];
                  const bool asc = (i & k) == 0;
                  if (asc ? (a > b) : (a < b)) {
                    ms.byid[i] = b;
                    ms.byid[ixj] = a;
                  }
                }
              }
              __syncwarp();
            }
          double a = 0.0;
          for (int i = lane; i < n3; i += 32) a += ms.wv[i];
          W = warp_sum_d(a);
          const double u = philox_uniform(seed, p.request_id, step);
          const double target = u * W;
          int pick = -1;
          double run = 0.0;
          for (int base = 0; base < n3 && pick < 0; base += 32) {
            const int i = base + lane;
            const double x = (i < n3) ? ms.wv[(uint32_t)ms.byid[i]] : 0.0;
            const double c = run + warp_incl_scan_d(x, lane);
            const unsigned hit = __ballot_sync(kFull, (i < n3) && (c > target));
            if (hit) pick = base + __ffs(hit) - 1;
            run = __shfl_sync(kFull, c, 31);
          }
          if (pick < 0) pick = n3 - 1;
          const int rank = (int)(uint32_t)ms.byid[pick];
          tok = comp_id(ms.top[rank]);
          lp = ((double)comp_val(ms.top[rank]) - (double)M) * inv_tau - log(S);
          flp = log(ms.wv[rank] / W);
        }
      }
    }
    if (lane == 0) {
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
        ro.logprobs[row] = (st == SAMPLER_ROW_OK) ? (float)lp : NAN;
        if (ro.flogprobs) ro.flogprobs[row] = (st == SAMPLER_ROW_OK) ? (float)flp : NAN;
        if (ro.status) ro.status[row] = st;
      }
    }
    __syncwarp();
    if (append && status == SAMPLER_ROW_OK) warp_append_token(hs, slot, tok, lane);
  }
  cbar();
}

}  // namespace smp

// merge.cuh — per-row merge of partial records and the final filter + draw (one warp per row).
//
// A row's partial records (pieces of one GPU's stream, or one record per vocab shard after the
// all-gather) carry (m, s, top-K candidates, frontier).  The merge combines
//     M = max m_i,   S = sum_i s_i * 2^((m_i - M) * log2(e)/tau)      (fixed order, float64)
// and the union of candidates (exact down to the max frontier), then applies — in the order
// of DESIGN.md R6 — top-k -> top-p (renormalised over the top-k survivors, R7/R8) -> min-p,
// and draws by inverse CDF over the kept set in ascending id order with a Philox uniform
// (R10, R11).  Candidate weights w_i = exp((z'_i - M)/tau) are float64.
#pragma once
#include "common.cuh"
#include "philox.cuh"
#include "warp_cand.cuh"

namespace smp {

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

// Incremental penalty-table update for one appended token ("only the B elements of f
// that correspond to the newly generated token IDs are incrementally updated").  One warp.
__device__ __forceinline__ void warp_append_token(const HistState& hs, int slot, int32_t tok,
                                                  int lane) {
  SlotMeta* sm = hs.meta + slot;
  const int np = sm->n_prompt, no = sm->n_out, nu = sm->n_uniq;
  if (np + no + 1 > hs.L) {
    if (lane == 0) sm->flags |= 1;
    return;
  }
  UniqEntry* u = hs.uniq + (int64_t)slot * hs.L;
  // lower_bound(tok) over ids (warp-parallel: count entries < tok)
  int less = 0;
  for (int i = lane; i < nu; i += 32) less += (u[i].id < tok) ? 1 : 0;
  less = warp_sum_i(less);
  const bool found = (less < nu) && (u[less].id == tok);
  __syncwarp();
  if (found) {
    if (lane == 0) u[less].meta += 2u;
  } else {
    // shift [less, nu) up by one, top block first
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

// Merge `nrec` records (pitch `rec_pitch` bytes, first at `recs`) of one row.
// mode 0: final decision + outputs (+ append).  mode 1: write one merged record to `out_rec`.
// Returns nothing; all lanes participate.  `w` supplies the warp's smem buffers.
__device__ __noinline__ void warp_merge_row(const uint8_t* recs, int64_t rec_pitch, int nrec,
                                            int row, int slot, const sampling_params& p,
                                            uint64_t seed, uint64_t step, int V, int kcand,
                                            int mode, uint8_t* out_rec, const RowOut& ro,
                                            int append, const HistState& hs, int lane,
                                            WarpCand& w, bool pending_ok) {
  const RowCfg rc = decode_row(p, V, kcand);
  // ---- headers
  float mloc = -INFINITY;
  int badloc = 0;
  uint64_t floc = 0;
  for (int i = lane; i < nrec; i += 32) {
    const RecHdr* h = reinterpret_cast<const RecHdr*>(recs + (int64_t)i * rec_pitch);
    mloc = fmaxf(mloc, h->m);
    badloc |= (h->flags & kRecBad) ? 1 : 0;
    floc = h->frontier > floc ? h->frontier : floc;
  }
  const float M = warp_max(mloc);
  const bool bad = __any_sync(kFull, badloc);
  uint64_t F = warp_max_u64(floc);
  double sloc = 0.0;
  for (int i = lane; i < nrec; i += 32) {
    const RecHdr* h = reinterpret_cast<const RecHdr*>(recs + (int64_t)i * rec_pitch);
    if (h->s != 0.0) sloc += h->s * exp2(((double)h->m - (double)M) * rc.c_d);
  }
  const double S = warp_sum_d(sloc);
  // ---- union of candidates, kept to the row's K
  w.reset(rc.keff);
  uint64_t thc = 0;  // composite admission threshold (current K-th once full)
  for (int i = 0; i < nrec; ++i) {
    const RecHdr* h = reinterpret_cast<const RecHdr*>(recs + (int64_t)i * rec_pitch);
    const uint64_t* e = reinterpret_cast<const uint64_t*>(h + 1);
    const int n = (int)h->n;
    for (int base = 0; base < n; base += 32) {
      const int j = base + lane;
      uint64_t v[1];
      int np = 0;
      if (j < n) {
        v[0] = e[j];
        np = v[0] >= thc ? 1 : 0;
      }
      warp_push<1>(w, v, np, lane);
      if (w.dropped) thc = make_comp(w.theta, 0x7FFFFFFF);  // conservative: value-level bound
    }
  }
  if (w.cnt > w.keff) warp_shrink(w, lane);
  int n = w.cnt;
  if (w.dropped && n > 0) {
    uint64_t mn = ~0ull;
    for (int i = lane; i < n; i += 32) mn = w.buf[i] < mn ? w.buf[i] : mn;
    mn = warp_min_u64(mn);
    F = mn > F ? mn : F;
  }

  if (mode == 1) {  // ---- local merge: emit one record
    RecHdr* oh = reinterpret_cast<RecHdr*>(out_rec);
    uint64_t* oe = reinterpret_cast<uint64_t*>(oh + 1);
    for (int i = lane; i < n; i += 32) oe[i] = w.buf[i];
    if (lane == 0) {
      RecHdr h;
      h.m = M;
      h.flags = bad ? kRecBad : 0u;
      h.s = S;
      h.n = (uint32_t)n;
      h.rsv = 0;
      h.frontier = F;
      *oh = h;
    }
    __syncwarp();
    return;
  }

  // ---- final decision
  int status = SAMPLER_ROW_OK;
  if (bad)
    status = SAMPLER_ROW_NONFINITE;
  else if (n == 0 || !(M > -INFINITY))
    status = SAMPLER_ROW_ALL_NEG_INF;
  int32_t tok = -1;
  double lp = NAN, flp = NAN, W = 0.0;
  uint64_t cutoff = 0;
  if (status == SAMPLER_ROW_OK) {
    warp_sort_desc(w.buf, n, lane);
    int n_exact = 0;
    for (int i = lane; i < n; i += 32) n_exact += (w.buf[i] >= F) ? 1 : 0;
    n_exact = warp_sum_i(n_exact);
    const bool complete = (F == 0);
    double* wv = reinterpret_cast<double*>(w.buf + 256);  // scratch after the <=128 entries
    const double inv_tau = 1.0 / (double)rc.tau;
    for (int i = lane; i < n; i += 32) wv[i] = exp(((double)comp_val(w.buf[i]) - (double)M) * inv_tau);
    __syncwarp();
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
          for (int i = lane; i < n1; i += 32) a += wv[i];
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
            const double x = (i < lim) ? wv[i] : 0.0;
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
          const unsigned hit = __ballot_sync(kFull, (i < n_exact) && (wv[i] < (double)rc.min_p));
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
      cutoff = w.buf[n3 - 1];
      if (rc.greedy) {
        tok = comp_id(w.buf[0]);
        W = 1.0;
        lp = ((double)comp_val(w.buf[0]) - (double)M) - log(S);
        flp = 0.0;
      } else {
        // draw: kept set K3 = first n3 of pi, walked in ascending id order (R10)
        uint64_t* byid = w.buf + 384;  // (id << 32 | rank)
        for (int i = lane; i < n3; i += 32)
          byid[i] = ((uint64_t)(uint32_t)comp_id(w.buf[i]) << 32) | (uint32_t)i;
        __syncwarp();
        warp_sort_asc(byid, n3, lane);
        double a = 0.0;
        for (int i = lane; i < n3; i += 32) a += wv[i];
        W = warp_sum_d(a);
        const double u = philox_uniform(seed, p.request_id, step);
        const double target = u * W;
        int pick = -1;
        double run = 0.0;
        for (int base = 0; base < n3 && pick < 0; base += 32) {
          const int i = base + lane;
          const double x = (i < n3) ? wv[(uint32_t)byid[i]] : 0.0;
          const double c = run + warp_incl_scan_d(x, lane);
          const unsigned hit = __ballot_sync(kFull, (i < n3) && (c > target));
          if (hit) pick = base + __ffs(hit) - 1;
          run = __shfl_sync(kFull, c, 31);
        }
        if (pick < 0) pick = n3 - 1;
        const int rank = (int)(uint32_t)byid[pick];
        tok = comp_id(w.buf[rank]);
        lp = ((double)comp_val(w.buf[rank]) - (double)M) * inv_tau - log(S);
        flp = log(wv[rank] / W);
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

}  // namespace smp

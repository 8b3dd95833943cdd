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

// Per-slot history state.  pmask[slot] is the slot's penalty presence bitmap (the set of ids in
// prompt u output — the support of the paper's penalty buffers f, kept as bits and
// updated incrementally on append) in phase A's step-lane order: local element le, v = le / vec,
// step k = v / 128, d = v % 128  ->  word k * 32 + (d % 32), bit (d / 32) * vec + le % vec.
// Phase A bulk-copies the words of each tile next to the logits and masks those elements.
struct HistState {
  SlotMeta* meta;
  UniqEntry* uniq;
  int32_t* tokens;
  int L;
  uint32_t* pmask;  // [max_batch][spr * 32]
  int spr;          // steps per row of the local slice
  int vec;          // elements per 16-byte vector (8 bf16 / 4 f32)
  int voff, vloc;
  int nslots;       // B_max
};

// Row r's request slot, validated on the device (device slot arrays are not checked on the host):
// an out-of-range slot reads slot 0 for memory safety and marks the row invalid.
__device__ __forceinline__ int row_slot(const int32_t* slots, int r, int nslots, bool* ok) {
  const int s = slots ? slots[r] : r;
  const bool v = s >= 0 && s < nslots;
  if (ok) *ok = v;
  return v ? s : 0;
}
// The parameter checks of sampler_set_params (R5), for device-supplied parameter arrays.
__device__ __forceinline__ bool params_ok(const sampling_params& p, int pen_mode) {
  if (!(p.temperature >= 0.0f) || !(p.temperature < INFINITY)) return false;
  if (!(p.top_p > 0.0f && p.top_p <= 1.0f)) return false;
  if (!(p.min_p >= 0.0f && p.min_p <= 1.0f)) return false;
  if (!(fabsf(p.repetition_penalty) < INFINITY) || !(fabsf(p.presence_penalty) < INFINITY) ||
      !(fabsf(p.frequency_penalty) < INFINITY))
    return false;
  if (pen_mode == SAMPLER_PEN_OPENAI_CTRL && !(p.repetition_penalty > 0.0f)) return false;
  return p.reserved == 0;
}

__host__ __device__ inline void pmask_pos(int le, int vec, int* word, uint32_t* bit) {
  const int v = le / vec, k = v / 128, d = v % 128;
  *word = k * 32 + (d & 31);
  *bit = 1u << ((d >> 5) * vec + le % vec);
}

// a token entered the slot's history: its presence bit (idempotent)
__device__ __forceinline__ void pmask_set(const HistState& hs, int slot, int32_t tok) {
  const int le = tok - hs.voff;
  if (le < 0 || le >= hs.vloc) return;
  int w;
  uint32_t b;
  pmask_pos(le, hs.vec, &w, &b);
  atomicOr(hs.pmask + (int64_t)slot * hs.spr * 32 + w, b);
}

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
    if (lane == 0) pmask_set(hs, slot, tok);
  }
  if (lane == 0) {
    hs.tokens[(int64_t)slot * hs.L + np + no] = tok;
    sm->n_out = no + 1;
    if (!found) sm->n_uniq = nu + 1;
  }
  __syncwarp();
}

// Append `tok` to a long history (more unique entries than phase B stages in smem) by the whole
// block (P:371 incremental update): the insertion point by a two-round 256-way search of the sorted
// table, then the entries above it moved up one slot in chunks of 4 per thread from the top down
// (every chunk read before any of it is written), the new entry, the token.
__device__ __noinline__ void block_append_global(const HistState& hs, int slot, int32_t tok) {
  const int tid = threadIdx.x, nt = blockDim.x;
  SlotMeta* sm = hs.meta + slot;
  const int np = sm->n_prompt, no = sm->n_out, nu = sm->n_uniq;
  if (np + no + 1 > hs.L) {
    if (tid == 0) sm->flags |= 1;
    return;
  }
  UniqEntry* u = hs.uniq + (int64_t)slot * hs.L;
  // round 1: samples at i = t * step; the count below tok is a prefix
  const int step = (nu + nt - 1) / nt;
  const int i1 = tid * step;
  const int c1 = __syncthreads_count(i1 < nu && u[i1].id < tok);
  const int base = c1 > 0 ? (c1 - 1) * step + 1 : 0;  // (entries below base are < tok)
  int c2 = 0;  // round 2: the step - 1 entries after the last sample below tok
  for (int o = 0; o < step; o += nt) {
    const int i2 = base + o + tid;
    c2 += __syncthreads_count(o + tid < step && i2 < nu && u[i2].id < tok);
  }
  const int less = c1 > 0 ? base + c2 : 0;
  const bool found = less < nu && u[less].id == tok;
  if (found) {
    if (tid == 0) u[less].meta += 2u;
  } else {
    for (int top = nu; top > less; top -= 4 * nt) {
      UniqEntry e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = top - 1 - tid - q * nt;
        if (i >= less) e[q] = u[i];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = top - 1 - tid - q * nt;
        if (i >= less) u[i + 1] = e[q];
      }
      __syncthreads();
    }
    if (tid == 0) {
      UniqEntry e;
      e.id = tok;
      e.meta = 2u;
      u[less] = e;
      pmask_set(hs, slot, tok);
    }
  }
  if (tid == 0) {
    hs.tokens[(int64_t)slot * hs.L + np + no] = tok;
    sm->n_out = no + 1;
    if (!found) sm->n_uniq = nu + 1;
  }
}

// Final decision for one row by one warp (R6-R11): top-k -> top-p (renormalised over
// the top-k survivors) -> min-p over the candidates top[0..n) (sorted by pi), exact down to the
// frontier F; inverse-CDF draw over the kept set in ascending id order with the Philox uniform;
// outputs + RowInfo.  Returns the sampled token when the row's status is OK, else -1.
// Candidates live in registers (candidate i = lane + 32q); the id-order cumulative mass of each
// kept candidate is accumulated by broadcasting every kept (id, w) once — no sort, no barrier.
__device__ __forceinline__ int warp_decide(const MergeSmem& ms, int n, float M, double S, uint64_t F, bool bad,
                                        bool invalid,
                                        const RowCfg& rc, const sampling_params& p, uint64_t seed, uint64_t step,
                                        int row, const RowOut& ro, bool pending_ok, uint64_t* tr) {
  constexpr int Q = SAMPLER_KCAND_MAX / 32;
  constexpr int UNK = 0x7FFFFFFF;
  const int lane = threadIdx.x & 31;
#define DTR(k)                             \
  do {                                     \
    if (tr && lane == 0) tr[k] = gtimer(); \
  } while (0)
  DTR(8);
  const double inv_tau = 1.0 / (double)rc.tau;
  const uint64_t* top = ms.top;
  uint64_t c[Q];
  double w[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = lane + 32 * q;
    c[q] = (i < n) ? top[i] : 0ull;
    w[q] = (i < n && !rc.greedy) ? exp(((double)comp_val(c[q]) - (double)M) * inv_tau) : 0.0;
  }
  DTR(9);
  int status = SAMPLER_ROW_OK;
  if (invalid)
    status = SAMPLER_ROW_INVALID;
  else if (bad)
    status = SAMPLER_ROW_NONFINITE;
  else if (n == 0 || !(M > -INFINITY))
    status = SAMPLER_ROW_ALL_NEG_INF;
  int32_t tok = -1;
  double lp = NAN, flp = NAN, W = 0.0;
  uint64_t cutoff = 0;
  if (status == SAMPLER_ROW_OK) {
    int n_exact = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) n_exact += __popc(__ballot_sync(kFull, lane + 32 * q < n && c[q] >= F));
    const bool complete = (F == 0);
    int n3 = -1;
    if (rc.greedy) {
      n3 = (n_exact >= 1) ? 1 : -1;  // the top candidate must be certified (F)
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
      if (rc.top_p < 1.0f) {
        double W1 = 0.0;
        bool w1k = false;
        if (n1 != UNK) {
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (lane + 32 * q < n1) a += w[q];
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
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            if (32 * q >= lim || n2 != UNK) break;  // (uniform)
            const int i = lane + 32 * q;
            const double cq = run + warp_incl_scan_d((i < lim) ? w[q] : 0.0, lane);
            const unsigned hit = __ballot_sync(kFull, (i < lim) && (cq >= target));
            if (hit && n2 == UNK) n2 = 32 * q + __ffs(hit);
            run = __shfl_sync(kFull, cq, 31);
          }
          if (n2 == UNK && n1 != UNK && n1 <= n_exact) n2 = n1;  // rounding shortfall
          if (n2 != UNK) cand = cand < n2 ? cand : n2;
        }
      }
      DTR(10);
      if (ok && rc.min_p > 0.0f) {
        int nm = UNK;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const unsigned hit = __ballot_sync(kFull, (lane + 32 * q < n_exact) && (w[q] < (double)rc.min_p));
          if (hit && nm == UNK) nm = 32 * q + __ffs(hit) - 1;
        }
        if (nm == UNK && complete) nm = n;
        if (nm != UNK) cand = cand < nm ? cand : nm;
      }
      if (ok && cand != UNK && cand <= n_exact && cand >= 1) n3 = cand;
    }
    DTR(11);
    if (n3 < 0) {
      status = kRowPending;
    } else {
      cutoff = __shfl_sync(kFull, c[0], 0);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const uint64_t cc = __shfl_sync(kFull, c[q], (n3 - 1) & 31);
        if (q == (n3 - 1) >> 5) cutoff = cc;
      }
      if (rc.greedy) {
        const uint64_t c0 = __shfl_sync(kFull, c[0], 0);
        tok = comp_id(c0);
        W = 1.0;
        lp = ((double)comp_val(c0) - (double)M) - log(S);
        flp = 0.0;
      } else {
        // kept set K3 = first n3 of pi; the draw walks it in ascending id order (R10): every
        // kept candidate's id-rank (integer walk over the kept ids, smem broadcast), weights
        // placed in id order, one prefix scan, first cumulative mass > u*W
        int id[Q], rk[Q];
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const bool kept = lane + 32 * q < n3;
          id[q] = kept ? comp_id(c[q]) : 0x7FFFFFFF;
          rk[q] = 0;
          if (kept) a += w[q];
        }
        W = warp_sum_d(a);
        const double u = philox_uniform(seed, p.request_id, step);
        const double target = u * W;
        DTR(12);
        if (n3 <= 32) {
#pragma unroll 4
          for (int j = 0; j < n3; ++j) rk[0] += (comp_id(top[j]) < id[0]) ? 1 : 0;
        } else {
#pragma unroll 4
          for (int j = 0; j < n3; ++j) {
            const int idj = comp_id(top[j]);
#pragma unroll
            for (int q = 0; q < Q; ++q) rk[q] += (idj < id[q]) ? 1 : 0;
          }
        }
        double* wid = reinterpret_cast<double*>(ms.byid);
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (lane + 32 * q < n3) wid[rk[q]] = w[q];
        __syncwarp();
        int pick = -1;
        double run = 0.0;
        for (int base = 0; base < n3 && pick < 0; base += 32) {
          const int i = base + lane;
          const double cq = run + warp_incl_scan_d((i < n3) ? wid[i] : 0.0, lane);
          const unsigned hit = __ballot_sync(kFull, (i < n3) && (cq > target));
          if (hit) pick = base + __ffs(hit) - 1;
          run = __shfl_sync(kFull, cq, 31);
        }
        if (pick < 0) pick = n3 - 1;  // u*W at the top of the mass: the last in id order
        DTR(13);
        double lpl = 0.0, flpl = 0.0;
        int own = 0, tl = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (lane + 32 * q < n3 && rk[q] == pick) {
            own = 1;
            tl = id[q];
            lpl = ((double)comp_val(c[q]) - (double)M) * inv_tau - log(S);
            flpl = log(w[q] / W);
          }
        const int src = __ffs(__ballot_sync(kFull, own)) - 1;
        tok = __shfl_sync(kFull, tl, src);
        lp = __shfl_sync(kFull, lpl, src);
        flp = __shfl_sync(kFull, flpl, src);
        DTR(14);
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
  DTR(15);
#undef DTR
  return (status == SAMPLER_ROW_OK) ? tok : -1;
}

// Merge `nrec` records (pitch `pitch` bytes, first at `recs`) of one row; all kBT threads.
// mode 0: final decision + outputs (+ append).  mode 1: write one merged record to out_rec.
// Latency-shaped: one global round trip brings every header and the first keff entries of every
// record (fixed stride keff in the pool) together with the slot's history state; the rank merge
// runs the per-list searches side by side; one barrier later warp 0 decides.
__device__ __noinline__ void block_merge_row(const uint8_t* recs, int64_t pitch, int nrec, int row, int slot,
                                             const sampling_params& p, uint64_t seed, uint64_t step, int V,
                                             int kcand, int mode, uint8_t* out_rec, const RowOut& ro, int append,
                                             const HistState& hs, bool pending_ok, bool invalid, const MergeSmem& ms,
                                             uint64_t* tr) {
#define MTR(k)                              \
  do {                                      \
    if (tr && threadIdx.x == 0) tr[k] = gtimer(); \
  } while (0)
  MTR(1);
  const RowCfg rc = decode_row(p, V, kcand);
  const int tid = threadIdx.x, lane = tid & 31;
  const int keff = rc.keff;
  const bool do_app = append && mode == 0 && !invalid;
  // ---- one round trip: headers, entries, history meta
  const int nslot = nrec * keff;  // <= kMaxRec * SAMPLER_KCAND_MAX == kPool
  for (int i = tid; i < nslot; i += kBT) {
    const int rr = i / keff;
    ms.pool[i] = rec_entries(recs + (int64_t)rr * pitch)[i - rr * keff];
  }
  if (tid < nrec) ms.hdr[tid] = *reinterpret_cast<const RecHdr*>(recs + (int64_t)tid * pitch);
  SlotMeta smeta = {0, 0, 0, 0};
  if (do_app) smeta = hs.meta[slot];
  cbar();
  MTR(2);
  // ---- the slot's unique-token table into registers (used by the append after the decision)
  constexpr int kUR = 4;
  const int nu = smeta.n_uniq;
  const bool reg_app = do_app && nu <= kBT * kUR;
  UniqEntry ue[kUR];
#pragma unroll
  for (int q = 0; q < kUR; ++q) {
    const int i = tid + q * kBT;
    ue[q].id = 0x7FFFFFFF;
    ue[q].meta = 0;
    if (reg_app && i < nu) ue[q] = hs.uniq[(int64_t)slot * hs.L + i];
  }
  // ---- rank merge: element q of list r has rank q + sum_{o != r} |{entries of o > c}|
  int U = 0;
  for (int o = 0; o < nrec; ++o) U += min((int)ms.hdr[o].n, keff);
  for (int i = tid; i < nslot; i += kBT) {
    const int rr = i / keff, q = i - rr * keff;
    if (q >= min((int)ms.hdr[rr].n, keff)) continue;
    const uint64_t c = ms.pool[i];
    int rank = q;
    for (int o = 0; o < nrec; ++o) {
      if (o == rr) continue;
      const int no = min((int)ms.hdr[o].n, keff);
      const uint64_t* L = ms.pool + o * keff;
      int pos = 0;
#pragma unroll
      for (int st = 128; st; st >>= 1)
        if (pos + st <= no && L[pos + st - 1] > c) pos += st;
      rank += pos;
    }
    if (rank < keff) ms.top[rank] = c;
  }
  // ---- M, S, frontier, flags (warp 0, fixed record order within the warp tree)
  if (tid < 32) {
    const bool has = lane < nrec;
    const RecHdr hd = has ? ms.hdr[lane] : RecHdr{};
    const float M = warp_max(has ? hd.m : -INFINITY);
    // R - RM with RM rounded first (no FMA contraction): contracted, the difference of two equal
    // products would be the product's rounding residual — ~1e22 for |M| ~ 1e38 — and S overflow
    const double RM = __dmul_rn((double)M, rc.c_d);
    const double term = (has && hd.s != 0.0) ? hd.s * exp2(__dsub_rn(hd.R, RM)) : 0.0;
    const double S = warp_sum_d(term);
    const uint64_t F = warp_max_u64(has ? hd.frontier : 0ull);
    const unsigned fl = __reduce_or_sync(kFull, has ? hd.flags : 0u);
    if (lane == 0) {
      ms.bs.f[0] = M;
      ms.bs.d[0] = S;
      ms.bs.u[0] = F;
      ms.bs.i[0] = (int)fl;
    }
  }
  cbar();
  MTR(3);
  const int n = U < keff ? U : keff;
  const float M = ms.bs.f[0];
  const double S = ms.bs.d[0];
  uint64_t F = ms.bs.u[0];
  if (U > keff && n > 0) F = ms.top[n - 1] > F ? ms.top[n - 1] : F;
  const bool bad = (ms.bs.i[0] & kRecBad) != 0;

  // ---- final decision (warp 0)
  if (tid < 32) {
    const int t = warp_decide(ms, n, M, S, F, bad, invalid, rc, p, seed, step, row, ro, pending_ok, tr);
    if (lane == 0) ms.bs.i[1] = t;
  }
  MTR(4);
  cbar();
  // ---- history append (P:371 incremental update), whole block; the table is in registers
  const int32_t tok = ms.bs.i[1];
  if (!do_app || tok < 0) return;
  if (!reg_app) {  // very long unique tables: one warp, chunked shift through global memory
    if (tid < 32) warp_append_token(hs, slot, tok, lane);
    return;
  }
  const int np = smeta.n_prompt, no = smeta.n_out;
  if (np + no + 1 > hs.L) {
    if (tid == 0) hs.meta[slot].flags |= 1;
    return;
  }
  int cl = 0;
#pragma unroll
  for (int q = 0; q < kUR; ++q) {
    const int i = tid + q * kBT;
    if (i < nu) cl += (ue[q].id < tok ? 1 : 0) + (ue[q].id == tok ? (1 << 20) : 0);
  }
  const int cs = block_sum_i(cl, ms.bs);
  const int less = cs & ((1 << 20) - 1);
  const bool found = (cs >> 20) != 0;
  UniqEntry* u = hs.uniq + (int64_t)slot * hs.L;
#pragma unroll
  for (int q = 0; q < kUR; ++q) {
    const int i = tid + q * kBT;
    if (i < nu) {
      if (found && i == less) u[i].meta = ue[q].meta + 2u;
      if (!found && i >= less) u[i + 1] = ue[q];
    }
  }
  if (tid == 0) {
    if (!found) {
      UniqEntry e;
      e.id = tok;
      e.meta = 2u;
      u[less] = e;
      pmask_set(hs, slot, tok);  // the id is penalised from the next step on (phase A's presence bitmap)
    }
    hs.tokens[(int64_t)slot * hs.L + np + no] = tok;
    SlotMeta m2 = smeta;
    m2.n_out = no + 1;
    if (!found) m2.n_uniq = nu + 1;
    hs.meta[slot] = m2;
  }
  MTR(5);
#undef MTR
}

// NEXT-2: one thread waits until every rank's flag for row r has reached sq (acquire; bounded by the
// handle's timeout); returns 1 on timeout
__device__ __noinline__ int exch_wait_row(const ExchPeers& x, int r, uint32_t sq) {
  const uint32_t* fl = reinterpret_cast<const uint32_t*>(x.bases[x.rank] + x.flags_off);
  const uint64_t t0 = gtimer();
  for (int q = 0; q < x.world; ++q)
    while ((int32_t)(ld_acquire_flag(fl + (int64_t)q * x.nslots + r, x.world > 1) - sq) < 0) {
      if (gtimer() - t0 > x.timeout_ns) return 1;
      __nanosleep(64);
    }
  return 0;
}
__device__ __forceinline__ void exch_timeout_row(const RowOut& ro, int r) {
  ro.tokens[r] = -1;
  ro.logprobs[r] = NAN;
  if (ro.flogprobs) ro.flogprobs[r] = NAN;
  if (ro.status) ro.status[r] = SAMPLER_ROW_EXCHANGE_TIMEOUT;
  RowInfo ri{};
  ri.status = SAMPLER_ROW_EXCHANGE_TIMEOUT;
  ro.info[r] = ri;
}

// Sharded phase 2: one CTA per row merges the row's per-rank candidate records (rank order,
// P:375) into the final sample.
struct MergeArgs {
  const uint8_t* records;   // gathered: world blocks of B records
  int64_t rec_stride;
  int64_t rank_pitch;       // bytes between ranks' blocks
  int world;
  int V, kcand;
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  const uint64_t* step_dev;  // nullable: the decode step read on the device
  int append;
  HistState hs;
  RowOut ro;
  uint64_t* trace;  // debug: per-row phase timestamps (32 per row), nullable
  int pen_mode;
  ExchPeers xp;     // xp.world > 0: records come from the one-shot peer exchange (NEXT-2)
};
constexpr int kMergeKernelSmem = kPool * 8 + 3 * SAMPLER_KCAND_MAX * 8 + kMaxRec * 48 + (kMaxRec + 1) * 4 + 12 + 512;

__global__ void __launch_bounds__(kBT, 2) merge_rows_kernel(const __grid_constant__ MergeArgs m) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int r = blockIdx.x;
  MergeSmem ms;
  ms.pool = reinterpret_cast<uint64_t*>(smem);
  ms.top = reinterpret_cast<uint64_t*>(smem + kPool * 8);
  ms.wv = reinterpret_cast<double*>(smem + kPool * 8 + SAMPLER_KCAND_MAX * 8);
  ms.byid = reinterpret_cast<uint64_t*>(smem + kPool * 8 + 2 * SAMPLER_KCAND_MAX * 8);
  uint8_t* rest = smem + kPool * 8 + 3 * SAMPLER_KCAND_MAX * 8;
  ms.hdr = reinterpret_cast<RecHdr*>(rest);
  ms.off = reinterpret_cast<int*>(rest + kMaxRec * 48);
  uint8_t* scr = rest + kMaxRec * 48 + (kMaxRec + 1) * 4 + 12;
  scr = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(scr) + 15) & ~(uintptr_t)15);
  ms.bs.f = reinterpret_cast<float*>(scr);
  ms.bs.d = reinterpret_cast<double*>(scr + 32);
  ms.bs.u = reinterpret_cast<uint64_t*>(scr + 96);
  ms.bs.i = reinterpret_cast<int*>(scr + 224);
  uint64_t* tr = m.trace ? m.trace + 32 * (int64_t)r : nullptr;
  bool slot_ok;
  const int slot = row_slot(m.slots, r, m.hs.nslots, &slot_ok);
  const sampling_params prm = m.params_dev ? m.params_dev[r] : m.params_tab[slot];
  const uint64_t seed = m.seeds ? m.seeds[r] : prm.seed;
  const uint8_t* recs = m.records;
  if (m.xp.world > 0) {  // NEXT-2: wait for every rank's flag of this row, then read the local copies
    // launched with programmatic dependent launch; the grid wait orders this rank's publishing kernel,
    // the flags the peers' records
    const ExchPeers& x = m.xp;
    griddep_wait();
    if (threadIdx.x == 0) {  // (one thread reads and advances the row's sequence number; the others
      const uint32_t sq = x.mseq[r] + 1;  //  take it from shared memory after the barrier)
      x.mseq[r] = sq;
      ms.bs.i[3] = (int)sq;
      ms.bs.i[2] = exch_wait_row(x, r, sq);
    }
    cbar();
    const uint32_t sq = (uint32_t)ms.bs.i[3];
    if (ms.bs.i[2]) {  // a peer never published: report the row, never hang the GPU
      if (threadIdx.x == 0) exch_timeout_row(m.ro, r);
      return;
    }
    recs = x.bases[x.rank] + (int64_t)(sq & 1) * x.par_pitch;
  }
  block_merge_row(recs + (int64_t)r * m.rec_stride, m.rank_pitch, m.world, r, slot, prm, seed, m.step_dev ? *m.step_dev : m.step, m.V,
                  m.kcand, 0, nullptr, m.ro, m.append, m.hs, false, !slot_ok || !params_ok(prm, m.pen_mode), ms, tr);
}

}  // namespace smp

// resolve.cuh — NEXT-1: vocab-sharded rows whose kept set is not bounded by the exchanged
// candidates (top-p-only / min-p-only / unfiltered rows, top_k > K_cand), resolved exactly by a
// distributed, mass-weighted radix select over the pi-order composite keys.
//
// The paper combines the t logits shards B x V/t of a TP lm_head without gathering the logits
// (§5.1 (3)); its filter is over the whole renormalised distribution (§2.1 eq.).
// A row the candidate merge (merge.cuh) cannot decide is finished here in ROUNDS.  Every round is
// one launch of resolve_kernel on every rank (one CTA per row) followed by the caller's
// all-gather of a fixed-size payload per row (sampler_resolve_bytes); every rank ingests the
// same gathered bytes with the same integer arithmetic, so the per-row state (ResState, one per
// batch row in the handle) stays identical on all ranks without any further agreement.
//
// Keys and masses.  composite c = key(z') << 32 | ~id orders elements by pi (z' desc, id asc,
// DESIGN.md R9) when compared as unsigned integers, larger first.  The elements of pi are those
// with float64 weight w = exp((z' - M)/tau) > 0 (the oracle's order_pi).  Masses are exchanged as
// 128-bit fixed point, w * 2^80 truncated (w <= 1, sums < 2^111): integer sums are exact and
// order-independent, so every rank derives the same cumulative masses; a mass is compared with a
// float64 target only after one monotone conversion (to_d).  The truncation (< 2^-80 per element)
// is far inside the 1e-10 * W parity band (R16).
//
// Per row, the state machine (phase) and what its payload carries:
//   K   top-k cutoff: the k-th element of pi.        payload: a 256-bin histogram (count, mass) of the
//   P   top-p cutoff: the first pi prefix whose      elements in the current key interval, bins =
//       cumulative mass >= p * W1 (W1 = mass of the  the next 8 bits of (khi - c); or, once the target
//       top-k survivors; R7, R8)                     bin holds <= kResCap elements, the elements
//                                                    themselves (composites), sorted and walked exactly
//   TOT kept mass of this rank's slice (pi prefix >= cut, w >= min_p: R6)  -> W, u*W, the owner rank
//   RES the owner walks its slice in ascending id order (R10) -> token, logprob, filtered logprob
//   -> outputs (+ history append, replicated on every rank) -> DONE.
// A K or P search takes at most 8 histogram rounds + 1 gather round (8 bits of the 64-bit key per
// round); a row takes at most kResMaxRounds exchanges in total.
#pragma once
#include "elem.cuh"
#include "merge.cuh"
#include "piece.cuh"

namespace smp {

typedef unsigned __int128 u128;

constexpr int kResThreads = 512;
constexpr int kResW = kResThreads / 32;
constexpr int kResBins = 256;                                   // 8 bits of the composite per round
constexpr int kResBodyWords = kResBins / 2 + 2 * kResBins;      // counts (u32) + masses (u128)
constexpr int kResCap = kResBodyWords - 2;                      // composites per gather payload
constexpr int64_t kResRowBytes = 16 + 8 * (int64_t)kResBodyWords;
constexpr int kResMaxRounds = 20;                               // 2 x (8 hist + 1 gather) + TOT + RES
static_assert(kResRowBytes % 16 == 0, "payload rows are copied as 16-byte vectors");

enum { RPH_DONE = 0, RPH_K = 1, RPH_P = 2, RPH_TOT = 3, RPH_RES = 4 };
enum { RK_NONE = 0, RK_HIST = 1, RK_GATHER = 2, RK_TOT = 3, RK_RES = 4 };

struct ResHdr {
  uint32_t kind;  // RK_*
  uint32_t n;     // RK_GATHER: entries
  uint64_t rsv;
};

struct __align__(16) ResState {
  int32_t phase, mode, shift, owner;  // mode: RK_HIST | RK_GATHER while searching
  uint64_t klo, khi;                  // search interval of composites (inclusive)
  uint64_t bcnt;                      // elements of the domain above khi
  uint64_t bm_lo, bm_hi;              // their mass (u128)
  uint64_t cut;                       // kept = { c >= cut, w > 0 } (then min-p)
  uint64_t pre_lo, pre_hi;            // TOT -> RES: mass of the ranks before the owner
  double T;                           // P: p * W1 (NaN until the first P ingest)
  double W;                           // kept mass
  double target;                      // u * W
  double S;
  float M;
  int32_t last;                       // u*W at the very top of the mass: the last kept id wins
  uint64_t wlo[16], whi[16];          // TOT -> RES: kept mass of each warp's id range (this rank)
  uint32_t wcnt[16];
  int32_t wlast[16];
};

struct ResolveArgs {
  const uint8_t* logits;  // this rank's slice [B x ld]
  int64_t ld;             // elements
  int esize;
  int B, V, kcand;
  int world, rank, round;
  const uint8_t* gathered;  // world x (B x kResRowBytes), rank order (round > 0)
  uint8_t* payload;         // B x kResRowBytes (this rank's contribution to the next exchange)
  const int32_t* slots;
  const sampling_params* params_dev;
  const sampling_params* params_tab;
  const uint64_t* seeds;
  uint64_t step;
  const uint64_t* step_dev;  // nullable: the decode step read on the device
  int append;
  HistState hs;
  RowOut ro;
  const RowInfo* info;  // the merge's per-row M, S and status (round 0)
  ResState* rs;         // [B]
  int32_t* active;      // rows still unresolved after this round (nullable)
  int pen_mode;
  ExchPeers rx;         // rx.world > 0: payloads through the one-shot peer exchange (NEXT-2), not gathered
};

__device__ __forceinline__ double to_d(u128 x) {
  return ((double)(uint64_t)(x >> 64) * 18446744073709551616.0 + (double)(uint64_t)x) * 0x1p-80;
}
__device__ __forceinline__ u128 mk128(uint64_t lo, uint64_t hi) { return ((u128)hi << 64) | lo; }
// w in [0, 1] as w * 2^80, truncated (exact for w >= 2^-27; mantissa bits below 2^-80 dropped)
__device__ __forceinline__ u128 wfix(double w) {
  const uint64_t b = (uint64_t)__double_as_longlong(w);
  const int E = (int)(b >> 52) & 0x7FF;
  if (E == 0) return 0;
  const uint64_t mm = (b & ((1ull << 52) - 1)) | (1ull << 52);
  const int sh = E - 995;  // mm * 2^(E - 1075) * 2^80
  if (sh >= 0) return (u128)mm << sh;
  if (sh <= -53) return 0;
  return (u128)(mm >> -sh);
}
__device__ __forceinline__ void atom_add128(unsigned long long* lo, unsigned long long* hi, u128 v) {
  const unsigned long long vl = (unsigned long long)v;
  unsigned long long vh = (unsigned long long)(v >> 64);
  const unsigned long long old = atomicAdd(lo, vl);
  if (old + vl < old) vh += 1;
  if (vh) atomicAdd(hi, vh);
}
// 64-bit shared add as two native 32-bit atomics with the carry (integer: order-independent)
__device__ __forceinline__ void smem_add_u64_32(uint64_t* p, uint64_t v) {
  uint32_t* p32 = reinterpret_cast<uint32_t*>(p);
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(p32, lo);
  const uint32_t up = hi + ((uint32_t)(old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(p32 + 1, up);
}
__device__ __forceinline__ u128 shfl_down128(u128 v, int o) {
  const uint64_t lo = __shfl_down_sync(kFull, (uint64_t)v, o);
  const uint64_t hi = __shfl_down_sync(kFull, (uint64_t)(v >> 64), o);
  return mk128(lo, hi);
}

struct ResRow {  // per-row constants of one round (smem)
  const uint8_t* rowp;
  const UniqEntry* uniq;
  const uint32_t* pm;
  int nu, slot;
  double M, tau, inv_tau, minp;
  sampling_params prm;
};

// z' of local element le (penalties through the slot's presence bitmap + sorted unique table)
template <typename T>
__device__ __forceinline__ float res_zp(const ResRow& r, const HistState& hs, int le, int pen_mode) {
  const float x = Dec<T>::load1(r.rowp, le);
  if (r.nu == 0) return x;
  int word;
  uint32_t bit;
  pmask_pos(le, hs.vec, &word, &bit);
  if (!(__ldg(r.pm + word) & bit)) return x;
  const int32_t id = hs.voff + le;
  int lo = 0, hi = r.nu;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (r.uniq[mid].id < id) lo = mid + 1;
    else hi = mid;
  }
  if (lo < r.nu && r.uniq[lo].id == id) return apply_penalty(x, r.uniq[lo].meta, r.prm, pen_mode);
  return x;
}
__device__ __forceinline__ double res_w(float z, const ResRow& r) { return exp(((double)z - r.M) * r.inv_tau); }

// z' of element t of local vector v (loaded as u, its presence bits pb)
template <typename T>
__device__ __forceinline__ float res_elem(const ResRow& r, const HistState& hs, const uint4 u, uint32_t pb, int v, int t,
                                          int pen_mode) {
  float z = Dec<T>::elem(u, t);
  if ((pb >> t) & 1u) {
    const int32_t id = hs.voff + v * Dec<T>::N + t;
    int lo = 0, hi = r.nu;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (r.uniq[mid].id < id) lo = mid + 1;
      else hi = mid;
    }
    if (lo < r.nu && r.uniq[lo].id == id) z = apply_penalty(z, r.uniq[lo].meta, r.prm, pen_mode);
  }
  return z;
}
template <typename T>
__device__ __forceinline__ uint32_t res_pbits(const ResRow& r, int v) {
  constexpr int VEC = Dec<T>::N;
  if (!r.nu) return 0u;
  const int k = v / 128, d = v % 128;
  return (__ldg(r.pm + k * 32 + (d & 31)) >> ((d >> 5) * VEC)) & ((1u << VEC) - 1u);
}

// z' of the elements of local vector v (16 bytes: 8 bf16 / 4 f32), in id order: fn(z', local id);
// penalised ids through the vector's bits of the slot's presence bitmap, then the sorted table
template <typename T, typename Fn>
__device__ __forceinline__ void res_vec(const ResRow& r, const HistState& hs, int v, int vloc, int pen_mode, Fn&& fn) {
  constexpr int VEC = Dec<T>::N;
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(r.rowp) + v);
  uint32_t pb = 0;
  if (r.nu) {
    const int k = v / 128, d = v % 128;
    pb = (__ldg(r.pm + k * 32 + (d & 31)) >> ((d >> 5) * VEC)) & ((1u << VEC) - 1u);
  }
#pragma unroll
  for (int t = 0; t < VEC; ++t) {
    const int le = v * VEC + t;
    if (le >= vloc) break;
    float z = Dec<T>::elem(u, t);
    if ((pb >> t) & 1u) {
      const int32_t id = hs.voff + le;
      int lo = 0, hi = r.nu;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (r.uniq[mid].id < id) lo = mid + 1;
        else hi = mid;
      }
      if (lo < r.nu && r.uniq[lo].id == id) z = apply_penalty(z, r.uniq[lo].meta, r.prm, pen_mode);
    }
    fn(z, le);
  }
}

struct ResSmem {
  ResState st;
  ResRow row;
  unsigned long long cnt[kResBins], mlo[kResBins], mhi[kResBins];
  uint32_t hc[kResBins];          // emission: counts (native 32-bit shared atomics)
  uint64_t hm[3][kResBins];       // emission: masses in three 27-bit pieces (each sum < 2^58)
  uint64_t ent[kResCap], srt[kResCap];
  uint64_t wlo[kResCap], whi[kResCap];
  uint64_t tlo[kResThreads + 1], thi[kResThreads + 1];
  uint32_t tcnt[kResThreads];
  int32_t tlast[kResThreads];
  int nent;
  int pick_le;
  const uint8_t* gbase;  // previous round's payloads (see res_rank_row)
  int64_t gpitch;
  uint8_t* outp;         // this round's payload of the row
  int timed_out;
  double pick_w;
  float pick_z;
};

// the previous round's payload of rank r for `row`: the caller's gathered buffer, or this rank's
// exchange region (parity of the previous publish) — g / pitch are set per CTA in the prologue
__device__ __forceinline__ const uint8_t* res_rank_row(const uint8_t* g, int64_t pitch, int r, int row) {
  return g + (int64_t)r * pitch + (int64_t)row * kResRowBytes;
}

// Start the P search over the domain { c >= lo } (W1 = the domain's mass, taken at the first ingest).
__device__ __forceinline__ void res_start_search(ResState& st, int phase, uint64_t lo) {
  st.phase = phase;
  st.mode = RK_HIST;
  st.shift = 56;
  st.klo = lo;
  st.khi = ~0ull;
  st.bcnt = 0;
  st.bm_lo = st.bm_hi = 0;
  st.T = NAN;
}
__device__ __forceinline__ void res_after_search(ResState& st, uint64_t cut, const sampling_params& p) {
  st.cut = cut;
  if (st.phase == RPH_K && p.top_p < 1.0f) res_start_search(st, RPH_P, cut);
  else st.phase = RPH_TOT;
}

template <typename T>
__global__ void __launch_bounds__(kResThreads, 1) resolve_kernel(const __grid_constant__ ResolveArgs a) {
  __shared__ ResSmem sm;
  const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  bool slot_ok;
  const int slot = row_slot(a.slots, row, a.hs.nslots, &slot_ok);
  const sampling_params prm = a.params_dev ? a.params_dev[row] : a.params_tab[slot];
  ResState& st = sm.st;
  if (tid == 0) {
    if (a.round == 0) {
      ResState s0{};
      const RowInfo ri = a.info[row];
      s0.phase = RPH_DONE;
      if (ri.status == kRowPending) {
        const RowCfg rc = decode_row(prm, a.V, a.kcand);
        s0.M = ri.M;
        s0.S = ri.S;
        if (rc.topk_on) res_start_search(s0, RPH_K, 0);
        else if (prm.top_p < 1.0f) res_start_search(s0, RPH_P, 0);
        else {
          s0.phase = RPH_TOT;
          s0.cut = 0;
        }
      }
      st = s0;
    } else {
      st = a.rs[row];
    }
    ResRow& r = sm.row;
    r.rowp = a.logits + (int64_t)row * a.ld * a.esize;
    r.slot = slot;
    r.nu = a.hs.meta[slot].n_uniq;
    r.uniq = a.hs.uniq + (int64_t)slot * a.hs.L;
    r.pm = a.hs.pmask + (int64_t)slot * a.hs.spr * 32;
    r.M = (double)st.M;
    r.tau = (double)decode_row(prm, a.V, a.kcand).tau;
    r.inv_tau = 1.0 / r.tau;
    r.minp = (double)prm.min_p;
    r.prm = prm;
  }
  if (tid == 0) {
    sm.timed_out = 0;
    const ExchPeers& x = a.rx;
    if (x.world == 0) {
      sm.gbase = a.gathered;
      sm.gpitch = (int64_t)a.B * kResRowBytes;
      sm.outp = a.payload + (int64_t)row * kResRowBytes;
    } else {
      // peer exchange: every rank published the previous round's payload of this row with sequence
      // number rq = x.seq[row] into every rank's region (parity rq & 1); wait for all of them
      const uint32_t rq = x.seq[row];
      uint8_t* own = x.bases[x.rank] + x.region_off;
      if (a.round > 0 && st.phase != RPH_DONE) {
        const uint32_t* fl = reinterpret_cast<const uint32_t*>(own + x.flags_off);
        const uint64_t t0 = gtimer();
        for (int q = 0; q < x.world && !sm.timed_out; ++q)
          while ((int32_t)(ld_acquire_flag(fl + (int64_t)q * x.nslots + row, x.world > 1) - rq) < 0) {
            if (gtimer() - t0 > x.timeout_ns) {
              sm.timed_out = 1;
              break;
            }
            __nanosleep(64);
          }
      }
      sm.gbase = own + (int64_t)(rq & 1) * x.par_pitch;
      sm.gpitch = x.rank_pitch;
      sm.outp = own + (int64_t)((rq + 1) & 1) * x.par_pitch + (int64_t)x.rank * x.rank_pitch +
                (int64_t)row * kResRowBytes;
    }
    if (sm.timed_out) {  // a peer stopped: report the row, never hang the GPU
      a.ro.tokens[row] = -1;
      a.ro.logprobs[row] = NAN;
      if (a.ro.flogprobs) a.ro.flogprobs[row] = NAN;
      if (a.ro.status) a.ro.status[row] = SAMPLER_ROW_EXCHANGE_TIMEOUT;
      st.phase = RPH_DONE;
      a.rs[row] = st;
    }
  }
  __syncthreads();
  if (st.phase == RPH_DONE) {
    if (tid == 0) {
      if (a.round == 0) a.rs[row] = st;
      if (a.rx.world == 0) reinterpret_cast<ResHdr*>(sm.outp)->kind = RK_NONE;
    }
    return;
  }
  const ResRow& R = sm.row;
  const int vloc = a.hs.vloc;
  const int nvec = (vloc + Dec<T>::N - 1) / Dec<T>::N;  // 16-byte vectors of the slice (ld * esize % 16 == 0)

  // ================================================================ ingest the last exchange
  if (a.round > 0) {
    const int ph = st.phase;
    if ((ph == RPH_K || ph == RPH_P) && st.mode == RK_HIST) {
      if (tid < kResBins) {  // bin sums over the ranks (integers: order-free)
        unsigned long long c = 0;
        u128 m = 0;
        for (int r = 0; r < a.world; ++r) {
          const uint8_t* p = res_rank_row(sm.gbase, sm.gpitch, r, row) + 16;
          c += reinterpret_cast<const uint32_t*>(p)[tid];
          const uint64_t* mp = reinterpret_cast<const uint64_t*>(p + 4 * kResBins);
          m += mk128(mp[2 * tid], mp[2 * tid + 1]);
        }
        sm.cnt[tid] = c;
        sm.mlo[tid] = (uint64_t)m;
        sm.mhi[tid] = (uint64_t)(m >> 64);
      }
      __syncthreads();
      if (tid == 0) {
        u128 bm = mk128(st.bm_lo, st.bm_hi);
        if (ph == RPH_P && st.T != st.T) {  // first P round covers the whole domain: W1
          u128 tot = 0;
          for (int j = 0; j < kResBins; ++j) tot += mk128(sm.mlo[j], sm.mhi[j]);
          st.T = (double)prm.top_p * to_d(tot);
        }
        const uint64_t k = (uint64_t)prm.top_k;
        uint64_t bc = st.bcnt;
        int js = -1, jlast = -1;
        for (int j = 0; j < kResBins; ++j) {
          const uint64_t cj = sm.cnt[j];
          if (cj == 0) continue;
          jlast = j;
          const u128 mj = mk128(sm.mlo[j], sm.mhi[j]);
          const bool hit = (ph == RPH_K) ? (bc + cj >= k) : (to_d(bm + mj) >= st.T);
          if (hit) {
            js = j;
            break;
          }
          bc += cj;
          bm += mj;
        }
        if (js < 0 && ph == RPH_P && jlast >= 0) {  // rounding shortfall (cannot happen for p <= 1)
          js = jlast;
          bc -= sm.cnt[jlast];
          bm -= mk128(sm.mlo[jlast], sm.mhi[jlast]);
        }
        if (js < 0) {
          // K: fewer than k elements have w > 0 -> all of pi is kept (oracle top_k_set)
          res_after_search(st, st.klo, prm);
        } else {
          st.bcnt = bc;
          st.bm_lo = (uint64_t)bm;
          st.bm_hi = (uint64_t)(bm >> 64);
          const uint64_t nhi = st.khi - ((uint64_t)js << st.shift);
          const uint64_t span = (st.shift >= 64) ? ~0ull : ((1ull << st.shift) - 1);
          const uint64_t nlo = (nhi - st.klo > span) ? nhi - span : st.klo;
          st.khi = nhi;
          st.klo = nlo;
          if (sm.cnt[js] <= (unsigned long long)kResCap) st.mode = RK_GATHER;
          else st.shift -= 8;
        }
      }
      __syncthreads();
    } else if ((ph == RPH_K || ph == RPH_P) && st.mode == RK_GATHER) {
      if (tid == 0) {
        int n = 0;
        for (int r = 0; r < a.world; ++r) {
          const uint8_t* p = res_rank_row(sm.gbase, sm.gpitch, r, row);
          const int nr = (int)reinterpret_cast<const ResHdr*>(p)->n;
          const uint64_t* e = reinterpret_cast<const uint64_t*>(p + 16);
          for (int i = 0; i < nr && n < kResCap; ++i) sm.ent[n++] = e[i];
        }
        sm.nent = n;
      }
      __syncthreads();
      const int n = sm.nent;
      for (int i = tid; i < n; i += kResThreads) {  // rank sort, descending (composites are distinct)
        const uint64_t c = sm.ent[i];
        int rk = 0;
        for (int j = 0; j < n; ++j) rk += sm.ent[j] > c ? 1 : 0;
        sm.srt[rk] = c;
      }
      __syncthreads();
      if (ph == RPH_P) {
        for (int i = tid; i < n; i += kResThreads) {
          const u128 wf = wfix(res_w(comp_val(sm.srt[i]), R));
          sm.wlo[i] = (uint64_t)wf;
          sm.whi[i] = (uint64_t)(wf >> 64);
        }
        __syncthreads();
      }
      if (tid == 0) {
        int pick = n - 1;
        if (ph == RPH_K) {
          const int64_t i = (int64_t)prm.top_k - (int64_t)st.bcnt - 1;
          pick = (int)(i < 0 ? 0 : (i > n - 1 ? n - 1 : i));
        } else {
          u128 cum = mk128(st.bm_lo, st.bm_hi);
          for (int i = 0; i < n; ++i) {
            cum += mk128(sm.wlo[i], sm.whi[i]);
            if (to_d(cum) >= st.T) {
              pick = i;
              break;
            }
          }
        }
        res_after_search(st, n > 0 ? sm.srt[pick] : st.klo, prm);
      }
      __syncthreads();
    } else if (ph == RPH_TOT) {
      if (tid == 0) {
        u128 tot = 0;
        for (int r = 0; r < a.world; ++r) {
          const uint64_t* b = reinterpret_cast<const uint64_t*>(res_rank_row(sm.gbase, sm.gpitch, r, row) + 16);
          tot += mk128(b[0], b[1]);
        }
        st.W = to_d(tot);
        const uint64_t seed = a.seeds ? a.seeds[row] : prm.seed;
        st.target = philox_uniform(seed, prm.request_id, a.step_dev ? *a.step_dev : a.step) * st.W;
        u128 pre = 0;
        int owner = -1, lastr = 0;
        for (int r = 0; r < a.world; ++r) {
          const uint64_t* b = reinterpret_cast<const uint64_t*>(res_rank_row(sm.gbase, sm.gpitch, r, row) + 16);
          const u128 tr = mk128(b[0], b[1]);
          if (b[2] > 0) lastr = r;
          if (to_d(pre + tr) > st.target) {
            owner = r;
            break;
          }
          pre += tr;
        }
        st.last = owner < 0;
        if (owner < 0) {  // u*W at the top of the mass: the last kept id (oracle draw_from)
          owner = lastr;
          pre = 0;
        }
        st.owner = owner;
        st.pre_lo = (uint64_t)pre;
        st.pre_hi = (uint64_t)(pre >> 64);
        st.phase = RPH_RES;
      }
      __syncthreads();
    } else if (ph == RPH_RES) {
      if (tid == 0) {
        const uint8_t* p = res_rank_row(sm.gbase, sm.gpitch, st.owner, row);
        const ResHdr hd = *reinterpret_cast<const ResHdr*>(p);
        const uint64_t* b = reinterpret_cast<const uint64_t*>(p + 16);
        int32_t tok = -1;
        if (hd.kind == RK_RES) {
          tok = (int32_t)b[0];
          a.ro.tokens[row] = tok;
          a.ro.logprobs[row] = (float)__longlong_as_double((long long)b[1]);
          if (a.ro.flogprobs) a.ro.flogprobs[row] = (float)__longlong_as_double((long long)b[2]);
          if (a.ro.status) a.ro.status[row] = SAMPLER_ROW_OK;
        }
        sm.pick_le = tok;
        st.phase = RPH_DONE;
      }
      __syncthreads();
      if (a.append && slot_ok && sm.pick_le >= 0) block_append_global(a.hs, slot, sm.pick_le);
    }
  }

  // ================================================================ this round's payload
  uint8_t* out = sm.outp;
  ResHdr* oh = reinterpret_cast<ResHdr*>(out);
  uint64_t* ob = reinterpret_cast<uint64_t*>(out + 16);
  const int ph = st.phase;
  // TOT / RES: warp-contiguous id ranges (coalesced rounds of 32 vectors); vec_kept = the kept mass
  // of one vector (and, with `before`, the first element whose cumulative mass crosses u*W)
    const uint64_t cut = st.cut;
    const int Sw = ((nvec + kResW * 32 - 1) / (kResW * 32)) * 32;
    const int wv0 = wid * Sw, wv1 = min(nvec, wv0 + Sw);
    auto vec_kept = [&](int v, u128* m, uint32_t* n, int* lastle, const u128* before,
                        int* pick) {
      // kept mass of vector v (and, with `before`, the first element whose cumulative crosses u*W)
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(R.rowp) + v);
      const uint32_t pb = res_pbits<T>(R, v);
      u128 cum = before ? *before : (u128)0;
      for (int t = 0; t < Dec<T>::N; ++t) {
        const int le = v * Dec<T>::N + t;
        if (le >= vloc) break;
        const float z = res_elem<T>(R, a.hs, u, pb, v, t, a.pen_mode);
        if (make_comp(z, a.hs.voff + le) < cut) continue;
        const double w = res_w(z, R);
        if (!(w > 0.0) || w < R.minp) continue;
        const u128 f = wfix(w);
        *m += f;
        *n += 1;
        *lastle = le;
        if (before) {
          cum += f;
          if (*pick < 0 && to_d(cum) > st.target) *pick = le;
        }
      }
    };
  if ((ph == RPH_K || ph == RPH_P) && st.mode == RK_HIST) {
    for (int j = tid; j < kResBins; j += kResThreads) {
      sm.hc[j] = 0;
      sm.hm[0][j] = sm.hm[1][j] = sm.hm[2][j] = 0;
    }
    __syncthreads();
    const uint64_t klo = st.klo, khi = st.khi;
    const int sh = st.shift;
    // shared 64-bit atomics are compare-and-swap loops (they spin under the contention of the first
    // rounds, where most of the row falls into a few bins): counts as native 32-bit atomics, masses
    // as three 27-bit pieces, each accumulated by two native 32-bit atomics with the carry
    for (int v = tid; v < nvec; v += kResThreads)
      res_vec<T>(R, a.hs, v, vloc, a.pen_mode, [&](float z, int le) {
        const uint64_t c = make_comp(z, a.hs.voff + le);
        if (c < klo || c > khi) return;
        const double w = res_w(z, R);
        if (!(w > 0.0)) return;
        const int j = (int)((khi - c) >> sh);
        const u128 f = wfix(w);
        atomicAdd(&sm.hc[j], 1u);
        smem_add_u64_32(&sm.hm[0][j], (uint64_t)f & 0x7FFFFFFull);
        smem_add_u64_32(&sm.hm[1][j], (uint64_t)(f >> 27) & 0x7FFFFFFull);
        const uint64_t p2 = (uint64_t)(f >> 54);
        if (p2) smem_add_u64_32(&sm.hm[2][j], p2);
      });
    __syncthreads();
    for (int j = tid; j < kResBins; j += kResThreads) {
      const u128 m = (u128)sm.hm[0][j] + ((u128)sm.hm[1][j] << 27) + ((u128)sm.hm[2][j] << 54);
      reinterpret_cast<uint32_t*>(ob)[j] = sm.hc[j];
      ob[kResBins / 2 + 2 * j] = (uint64_t)m;
      ob[kResBins / 2 + 2 * j + 1] = (uint64_t)(m >> 64);
    }
    if (tid == 0) {
      oh->kind = RK_HIST;
      oh->n = 0;
    }
  } else if ((ph == RPH_K || ph == RPH_P) && st.mode == RK_GATHER) {
    if (tid == 0) sm.nent = 0;
    __syncthreads();
    const uint64_t klo = st.klo, khi = st.khi;
    for (int v = tid; v < nvec; v += kResThreads)
      res_vec<T>(R, a.hs, v, vloc, a.pen_mode, [&](float z, int le) {
        const uint64_t c = make_comp(z, a.hs.voff + le);
        if (c < klo || c > khi) return;
        if (!(res_w(z, R) > 0.0)) return;
        const int i = atomicAdd(&sm.nent, 1);
        if (i < kResCap) ob[i] = c;
      });
    __syncthreads();
    if (tid == 0) {
      oh->kind = RK_GATHER;
      oh->n = (uint32_t)min(sm.nent, kResCap);
    }
  } else if (ph == RPH_TOT) {
    u128 acc = 0;
    uint32_t kc = 0;
    int lastle = -1;
    for (int v = wv0 + lane; v < wv1; v += 32) vec_kept(v, &acc, &kc, &lastle, nullptr, nullptr);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc += shfl_down128(acc, o);
      kc += __shfl_down_sync(kFull, kc, o);
      lastle = max(lastle, __shfl_down_sync(kFull, lastle, o));
    }
    if (lane == 0) {
      st.wlo[wid] = (uint64_t)acc;
      st.whi[wid] = (uint64_t)(acc >> 64);
      st.wcnt[wid] = kc;
      st.wlast[wid] = lastle;
    }
    __syncthreads();
    if (tid == 0) {
      u128 t = 0;
      uint64_t n = 0;
      for (int w = 0; w < kResW; ++w) {
        t += mk128(st.wlo[w], st.whi[w]);
        n += st.wcnt[w];
      }
      ob[0] = (uint64_t)t;
      ob[1] = (uint64_t)(t >> 64);
      ob[2] = n;
      oh->kind = RK_TOT;
      oh->n = 0;
    }
  } else if (ph == RPH_RES) {
    if (st.owner != a.rank) {
      if (tid == 0) oh->kind = RK_NONE;
    } else {
      // the owner: kept mass per warp range (ascending id, coalesced rounds of 32 vectors), the warp
      // prefix from the mass of the ranks before; the warp holding u*W re-walks its range round by
      // round (warp scans), the crossing lane walks its vector's elements
      // (the warp totals of this rank's TOT pass, kept in the row state)
      if (lane == 0) {
        sm.tlo[wid] = st.wlo[wid];
        sm.thi[wid] = st.whi[wid];
        sm.tcnt[wid] = st.wcnt[wid];
        sm.tlast[wid] = st.wlast[wid];
      }
      if (tid == 0) {
        sm.pick_le = -1;
        sm.nent = -1;  // (the crossing warp)
      }
      __syncthreads();
      if (tid == 0) {  // warp prefix from the mass of the ranks before; the crossing warp
        u128 p = mk128(st.pre_lo, st.pre_hi);
        int lt = -1;
        for (int w = 0; w < kResW; ++w) {
          const u128 v = mk128(sm.tlo[w], sm.thi[w]);
          if (sm.nent < 0 && !st.last && sm.tcnt[w] > 0 && to_d(p + v) > st.target) {
            sm.nent = w;
            sm.tlo[kResW] = (uint64_t)p;
            sm.thi[kResW] = (uint64_t)(p >> 64);
          }
          p += v;
          if (sm.tcnt[w] > 0) lt = max(lt, sm.tlast[w]);
        }
        if (st.last || sm.nent < 0) sm.pick_le = lt;  // (u*W at the top of the mass: the last kept id)
      }
      __syncthreads();
      if (wid == sm.nent) {
        u128 P = mk128(sm.tlo[kResW], sm.thi[kResW]);
        int found = -1;
        for (int vb = wv0; vb < wv1 && found < 0; vb += 32) {
          const int v = vb + lane;
          u128 m = 0;
          uint32_t n = 0;
          int ll = -1;
          if (v < wv1) vec_kept(v, &m, &n, &ll, nullptr, nullptr);
          u128 incl = m;  // inclusive warp scan (u128)
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint64_t lo = __shfl_up_sync(kFull, (uint64_t)incl, o);
            const uint64_t hi = __shfl_up_sync(kFull, (uint64_t)(incl >> 64), o);
            if (lane >= o) incl += mk128(lo, hi);
          }
          const bool cross = n > 0 && to_d(P + incl - m) <= st.target && to_d(P + incl) > st.target;
          const unsigned bal = __ballot_sync(kFull, cross);
          if (bal) {
            int pk = -1;
            if (lane == __ffs(bal) - 1) {
              const u128 before = P + incl - m;
              u128 m2 = 0;
              uint32_t n2 = 0;
              int l2 = -1;
              vec_kept(v, &m2, &n2, &l2, &before, &pk);
              if (pk < 0) pk = l2;  // (rounding inside the vector: its last kept)
            }
            found = __shfl_sync(kFull, pk, __ffs(bal) - 1);
          }
          const uint64_t tl = __shfl_sync(kFull, (uint64_t)incl, 31), th = __shfl_sync(kFull, (uint64_t)(incl >> 64), 31);
          P += mk128(tl, th);
        }
        if (lane == 0) sm.pick_le = found >= 0 ? found : sm.tlast[wid];  // (rounding: the warp's last kept)
      }
      __syncthreads();
      if (tid == 0) {
        const int le = sm.pick_le;
        if (le >= 0) {
          const float z = res_zp<T>(R, a.hs, le, a.pen_mode);
          const double w = res_w(z, R);
          ob[0] = (uint64_t)(uint32_t)(a.hs.voff + le);
          ob[1] = (uint64_t)__double_as_longlong(((double)z - R.M) / R.tau - log(st.S));
          ob[2] = (uint64_t)__double_as_longlong(log(w / st.W));
          oh->kind = RK_RES;
        } else {
          oh->kind = RK_NONE;
        }
      }
    }
  } else if (tid == 0) {
    oh->kind = RK_NONE;
  }
  if (a.rx.world > 0 && st.phase != RPH_DONE) {
    // publish: the payload (written into this rank's own region above) copied into every peer's
    // region, then the row's flag raised everywhere (release after the CTA barrier)
    const ExchPeers& x = a.rx;
    __syncthreads();
    const int64_t off = out - x.bases[x.rank];
    constexpr int kN16 = (int)(kResRowBytes / 16);
    for (int p = 0; p < x.world; ++p) {
      if (p == x.rank) continue;
      uint4* dst = reinterpret_cast<uint4*>(x.bases[p] + off);
      const uint4* src = reinterpret_cast<const uint4*>(out);
      for (int i = tid; i < kN16; i += kResThreads) dst[i] = src[i];
    }
    if (x.world > 1) __threadfence_system();  // (each storing thread's own writes, before the release)
    else __threadfence();
    __syncthreads();
    if (tid == 0) {
      const uint32_t sq = x.seq[row] + 1;
      x.seq[row] = sq;
      for (int p = 0; p < x.world; ++p)
        st_release_flag(reinterpret_cast<uint32_t*>(x.bases[p] + x.region_off + x.flags_off) + (int64_t)x.rank * x.nslots + row,
                        sq, x.world > 1);
    }
  }
  if (tid == 0) {
    a.rs[row] = st;
    if (a.active && st.phase != RPH_DONE) atomicAdd(a.active, 1);
  }
}

}  // namespace smp

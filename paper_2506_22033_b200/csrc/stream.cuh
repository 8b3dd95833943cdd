// stream.cuh — the one-pass streaming kernel: logits [B x V] -> per-row samples.
//
// Work decomposition (B200-first; not the paper's CPU column layout):
//   the padded logits space [B x Vp] is flattened and cut into equal contiguous spans, one per
//   warp, across a persistent grid of 148 SMs x 2 CTAs x 8 warps.  Every warp streams its span
//   through a private 4-stage ring of 2 KB shared-memory tiles filled by 1-D bulk async copies
//   (cp.async.bulk, the TMA engine) — no block barriers anywhere.  Balance is exact at any B.
//   A span that crosses a row boundary yields one "piece" per row.  Per piece the warp keeps
//     * lane-private online max / sum of 2^((z' - m_ref) * log2(e)/tau)   (float64 accumulators)
//     * the piece's exact top-K candidates (warp_cand.cuh)
//   and penalties are applied by sparse scatter from the slot's incremental unique-token table
//    into the tile before it is read (penalised entries processed as scalars, then
//   replaced by a -inf sentinel).  Each piece writes a record; the LAST piece of a row to finish
//   (atomic ticket) merges the row's records (merge.cuh) — one launch per decode step.
//
// Per element: 1 shared-memory vector load / 8 elements, bf16->f32, 3 FP32 ops, 1 MUFU ex2, a
// pairwise add; one compare per vector against the admission threshold.  HBM bytes = the logits
// exactly once (+ the penalty table entries).
#pragma once
#include "common.cuh"
#include "merge.cuh"
#include "warp_cand.cuh"

namespace smp {

constexpr int kWarpsPerCta = 8;
constexpr int kStages = 4;
constexpr int kChunkBytes = 2048;
constexpr int kPerWarpSmem = kStages * kChunkBytes + kCapW * 8 + 256 * 4 + kStages * 8;
constexpr int kStreamSmem = kWarpsPerCta * kPerWarpSmem;

struct StreamArgs {
  const void* logits;
  int64_t ld;          // row stride (elements)
  int B;
  int V;               // global vocab
  int voff, vloc;      // local slice
  int Vp;              // vloc rounded up to the vector width
  int64_t span;        // elements per warp (multiple of the vector width)
  int64_t N;           // B * Vp
  const int32_t* slots;
  const sampling_params* params_dev;  // nullable
  const sampling_params* params_tab;
  const uint64_t* seeds;              // nullable
  uint64_t step;
  int append;
  int kcand;
  int pen_mode;
  HistState hs;
  uint8_t* records;
  int64_t rec_stride;
  int32_t* tickets;
  int mode;            // 0 final, 1 local (sharded phase 1)
  uint8_t* out_records;
  RowOut ro;
  int pending_ok;
};

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <typename T>
struct VecT;
template <>
struct VecT<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void load(const uint8_t* p, float (&z)[8], float& vmax) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&u.z);
    __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&u.w);
    const __nv_bfloat162 m = __hmax2_nan(__hmax2_nan(a, b), __hmax2_nan(c, d));
    vmax = fmax_nan(__low2float(m), __high2float(m));
    z[0] = __uint_as_float(u.x << 16);
    z[1] = __uint_as_float(u.x & 0xFFFF0000u);
    z[2] = __uint_as_float(u.y << 16);
    z[3] = __uint_as_float(u.y & 0xFFFF0000u);
    z[4] = __uint_as_float(u.z << 16);
    z[5] = __uint_as_float(u.z & 0xFFFF0000u);
    z[6] = __uint_as_float(u.w << 16);
    z[7] = __uint_as_float(u.w & 0xFFFF0000u);
  }
  static __device__ __forceinline__ float get(const uint8_t* tile, int j) {
    const uint16_t b = reinterpret_cast<const uint16_t*>(tile)[j];
    return __uint_as_float((uint32_t)b << 16);
  }
  static __device__ __forceinline__ void set_neg_inf(uint8_t* tile, int j) {
    reinterpret_cast<uint16_t*>(tile)[j] = 0xFF80u;
  }
};
template <>
struct VecT<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void load(const uint8_t* p, float (&z)[4], float& vmax) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    z[0] = u.x;
    z[1] = u.y;
    z[2] = u.z;
    z[3] = u.w;
    vmax = fmax_nan(fmax_nan(u.x, u.y), fmax_nan(u.z, u.w));
  }
  static __device__ __forceinline__ float get(const uint8_t* tile, int j) {
    return reinterpret_cast<const float*>(tile)[j];
  }
  static __device__ __forceinline__ void set_neg_inf(uint8_t* tile, int j) {
    reinterpret_cast<float*>(tile)[j] = -INFINITY;
  }
};

// Penalised logit, every op correctly rounded binary32 with no contraction (R1, R3).
__device__ __forceinline__ float apply_penalty(float x, uint32_t meta, const sampling_params& p,
                                               int mode) {
  const int cnt = (int)(meta >> 1);
  float y = x;
  if (mode == SAMPLER_PEN_OPENAI_CTRL) {
    const float r = p.repetition_penalty;
    if (r != 1.0f) y = (y > 0.0f) ? __fdiv_rn(y, r) : __fmul_rn(y, r);
    if (cnt > 0) {
      y = __fsub_rn(y, __fmul_rn(p.frequency_penalty, (float)cnt));
      y = __fsub_rn(y, p.presence_penalty);
    }
  } else {
    y = __fsub_rn(y, __fmul_rn(p.frequency_penalty, (float)cnt));
    y = __fsub_rn(y, cnt > 0 ? p.presence_penalty : 0.0f);
    y = __fsub_rn(y, p.repetition_penalty);
  }
  return y;
}

// lane-private online reduction state
struct LaneAcc {
  float mref;  // reference for the exponent (rescaled lazily, margin delta)
  float thr;   // mref + delta
  float mmax;  // exact max seen
  double acc;  // sum 2^((z - mref) * c)
  int bad;
};

__device__ __forceinline__ void lane_rescale(LaneAcc& a, float vmax, const RowCfg& rc) {
  if (a.acc != 0.0) a.acc *= exp2(((double)a.mref - (double)vmax) * rc.c_d);
  a.mref = vmax;
  a.thr = vmax + rc.delta;
}

template <typename T>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 2) stream_kernel(const StreamArgs a) {
  using VT = VecT<T>;
  constexpr int VEC = VT::N;
  constexpr int ESZ = (int)sizeof(T);
  constexpr int CH = kChunkBytes / ESZ;  // elements per chunk

  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + wib;
  const int64_t a0 = gw * a.span;
  const int64_t a1 = min(a.N, a0 + a.span);
  if (a0 >= a1) return;

  uint8_t* wsm = smem + wib * kPerWarpSmem;
  uint8_t* stage = wsm;
  WarpCand wc;
  wc.buf = reinterpret_cast<uint64_t*>(wsm + kStages * kChunkBytes);
  wc.hist = reinterpret_cast<uint32_t*>(wsm + kStages * kChunkBytes + kCapW * 8);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wsm + kStages * kChunkBytes + kCapW * 8 + 256 * 4);

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = l2_evict_first_policy();
  const uint8_t* lg = reinterpret_cast<const uint8_t*>(a.logits);

  // producer cursor (lane 0 only uses it)
  int64_t ppos = a0;
  auto issue = [&](int s) {
    if (ppos >= a1) return;
    const int64_t r = ppos / a.Vp;
    const int64_t off = ppos - r * a.Vp;
    int64_t len = a.Vp - off;
    if (len > CH) len = CH;
    if (len > a1 - ppos) len = a1 - ppos;
    const uint8_t* src = lg + (r * a.ld + off) * ESZ;
    mbar_arrive_expect_tx(&bars[s], (uint32_t)(len * ESZ));
    bulk_g2s(stage + s * kChunkBytes, src, (uint32_t)(len * ESZ), &bars[s], pol);
    ppos += len;
  };
  if (lane == 0)
    for (int s = 0; s < kStages; ++s) issue(s);

  // consumer state
  int64_t cpos = a0;
  int cur_r = -1;
  int slot = 0;
  sampling_params prm;
  RowCfg rc;
  LaneAcc la;
  int pc = 0, pend = 0;  // penalty cursor in the slot's unique table
  const UniqEntry* utab = nullptr;

  auto start_piece = [&](int r, int64_t off) {
    cur_r = r;
    slot = a.slots ? a.slots[r] : r;
    prm = a.params_dev ? a.params_dev[r] : a.params_tab[slot];
    rc = decode_row(prm, a.V, a.kcand);
    la.mref = -INFINITY;
    la.thr = -INFINITY;
    la.mmax = -INFINITY;
    la.acc = 0.0;
    la.bad = 0;
    wc.reset(rc.keff);
    // penalty entries with global id >= voff + off (lower_bound, warp-parallel count)
    utab = a.hs.uniq + (int64_t)slot * a.hs.L;
    const int nu = a.hs.meta[slot].n_uniq;
    const int lo = a.voff + (int)off;
    int less = 0;
    for (int i = lane; i < nu; i += 32) less += (utab[i].id < lo) ? 1 : 0;
    pc = warp_sum_i(less);
    pend = nu;
  };

  auto finish_piece = [&]() {
    const int r = cur_r;
    if (wc.cnt > wc.keff) warp_shrink(wc, lane);
    uint64_t fr = 0;
    if (wc.dropped) {
      uint64_t mn = ~0ull;
      for (int i = lane; i < wc.cnt; i += 32) mn = wc.buf[i] < mn ? wc.buf[i] : mn;
      fr = warp_min_u64(mn);
    }
    const float m = warp_max(la.mmax);
    double s = 0.0;
    if (la.acc != 0.0) s = la.acc * exp2(((double)la.mref - (double)m) * rc.c_d);
    s = warp_sum_d(s);
    const bool bad = __any_sync(kFull, la.bad);
    uint8_t* rec = a.records + (gw + r) * a.rec_stride;
    uint64_t* ent = reinterpret_cast<uint64_t*>(rec + sizeof(RecHdr));
    for (int i = lane; i < wc.cnt; i += 32) ent[i] = wc.buf[i];
    if (lane == 0) {
      RecHdr h;
      h.m = m;
      h.flags = bad ? kRecBad : 0u;
      h.s = s;
      h.n = (uint32_t)wc.cnt;
      h.rsv = 0;
      h.frontier = fr;
      *reinterpret_cast<RecHdr*>(rec) = h;
    }
    __threadfence();
    __syncwarp();
    const int64_t w_first = ((int64_t)r * a.Vp) / a.span;
    const int64_t w_last = ((int64_t)(r + 1) * a.Vp - 1) / a.span;
    const int npieces = (int)(w_last - w_first + 1);
    int last = 0;
    if (lane == 0) last = (atomicAdd(&a.tickets[r], 1) == npieces - 1);
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      __threadfence();
      const uint64_t seed = a.seeds ? a.seeds[r] : prm.seed;
      warp_merge_row(a.records + (w_first + r) * a.rec_stride, a.rec_stride, npieces, r, slot, prm,
                     seed, a.step, a.V, a.kcand, a.mode,
                     a.out_records ? a.out_records + (int64_t)r * a.rec_stride : nullptr, a.ro,
                     a.append, a.hs, lane, wc, a.pending_ok != 0);
      if (lane == 0) a.tickets[r] = 0;
    }
  };

  int it = 0;
  while (cpos < a1) {
    const int s = it % kStages;
    const uint32_t par = (uint32_t)((it / kStages) & 1);
    const int r = (int)(cpos / a.Vp);
    const int64_t off = cpos - (int64_t)r * a.Vp;
    int64_t len64 = a.Vp - off;
    if (len64 > CH) len64 = CH;
    if (len64 > a1 - cpos) len64 = a1 - cpos;
    const int len = (int)len64;
    if (r != cur_r) {
      if (cur_r >= 0) finish_piece();
      start_piece(r, off);
    }
    uint8_t* tile = stage + s * kChunkBytes;
    mbar_wait(&bars[s], par);

    // padding tail of the row (ids >= vloc): -inf
    if (off + len > a.vloc) {
      const int j0 = (int)(a.vloc - off) > 0 ? (int)(a.vloc - off) : 0;
      for (int j = j0 + lane; j < len; j += 32) VT::set_neg_inf(tile, j);
    }
    // ---- penalties: sparse scatter from the slot's unique-token table
    const int gid0 = a.voff + (int)off;
    const int gid1 = gid0 + (int)min((int64_t)len, (int64_t)a.vloc - off);  // no padding ids
    while (pc < pend) {
      const int i = pc + lane;
      UniqEntry e;
      bool in = false;
      if (i < pend) {
        e = utab[i];
        in = e.id < gid1;
      }
      const unsigned m = __ballot_sync(kFull, in);
      uint64_t cv[1];
      int np = 0;
      if (in) {
        const int j = e.id - gid0;
        const float x = VT::get(tile, j);
        la.bad |= !(x < INFINITY) ? 1 : 0;  // NaN or +inf raw logit
        const float y = apply_penalty(x, e.meta, prm, a.pen_mode);
        if (y > -INFINITY) {
          if (y > la.thr) lane_rescale(la, y, rc);
          const float t = y - la.mref;
          la.acc += (double)ex2f(fmaf(t, rc.c_hi, t * rc.c_lo));
          la.mmax = fmaxf(la.mmax, y);
          if (y >= wc.theta) {
            cv[0] = make_comp(y, e.id);
            np = 1;
          }
        }
        VT::set_neg_inf(tile, j);
      }
      __syncwarp();
      warp_push<1>(wc, cv, np, lane);
      const int nin = __popc(m);
      pc += nin;
      if (nin < 32) break;
    }
    __syncwarp();

    // ---- bulk: one 16-byte vector per lane per step
    const int nvec = len / VEC;
    for (int base = 0; base < nvec; base += 32) {
      const int v = base + lane;
      float z[VEC];
      float vmax = -INFINITY;
      bool want = false;
      if (v < nvec) {
        VT::load(tile + v * 16, z, vmax);
        la.bad |= !(vmax < INFINITY) ? 1 : 0;
        if (vmax > -INFINITY) {
          if (vmax > la.thr) lane_rescale(la, vmax, rc);
          float e[VEC];
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            const float t = z[i] - la.mref;
            e[i] = ex2f(fmaf(t, rc.c_hi, t * rc.c_lo));
          }
#pragma unroll
          for (int st = 1; st < VEC; st <<= 1)
#pragma unroll
            for (int i = 0; i < VEC; i += 2 * st) e[i] += e[i + st];
          la.acc += (double)e[0];
          la.mmax = fmaxf(la.mmax, vmax);
          want = vmax >= wc.theta;
        }
      }
      if (__any_sync(kFull, want)) {
        uint32_t msk = 0;
        if (want) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) msk |= (z[i] >= wc.theta) ? (1u << i) : 0u;
        }
        int total;
        int pos = warp_push_slot(wc, __popc(msk), lane, &total);
        const int id0 = gid0 + v * VEC;
#pragma unroll
        for (int i = 0; i < VEC; ++i)
          if (msk & (1u << i)) wc.buf[pos++] = make_comp(z[i], id0 + i);
        warp_push_done(wc, total, lane);
      }
    }
    __syncwarp();
    cpos += len;
    if (lane == 0) issue(s);
    ++it;
  }
  if (cur_r >= 0) finish_piece();
}

// Phase 2 of vocab-sharded sampling: one warp per row merges `world` rank records.
__global__ void __launch_bounds__(kWarpsPerCta * 32) merge_kernel(
    const uint8_t* gathered, int64_t rank_pitch, int64_t rec_stride, int world, int B,
    const int32_t* slots, const sampling_params* params_dev, const sampling_params* params_tab,
    const uint64_t* seeds, uint64_t step, int V, int kcand, int append, HistState hs, RowOut ro) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int r = blockIdx.x * kWarpsPerCta + wib;
  if (r >= B) return;
  WarpCand wc;
  wc.buf = reinterpret_cast<uint64_t*>(smem + wib * (kCapW * 8 + 1024));
  wc.hist = reinterpret_cast<uint32_t*>(smem + wib * (kCapW * 8 + 1024) + kCapW * 8);
  const int slot = slots ? slots[r] : r;
  const sampling_params prm = params_dev ? params_dev[r] : params_tab[slot];
  const uint64_t seed = seeds ? seeds[r] : prm.seed;
  warp_merge_row(gathered + (int64_t)r * rec_stride, rank_pitch, world, r, slot, prm, seed, step, V,
                 kcand, 0, nullptr, ro, append, hs, lane, wc, false);
}

}  // namespace smp

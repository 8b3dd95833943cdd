/* sampler_cpu.c -- the paper's own CPU sampling design as a comparator.
 *
 * NOT part of the product path (the product is the CUDA library behind include/sampler.h); this is
 * a baseline that bench.py times on the host cores beside the GPU number, so that the GPU-vs-CPU
 * sampling trade-off the paper makes (SiPipe section 5.1) is measured against
 * the paper's design rather than against the deliberately slow float64 oracle.
 *
 * What it follows from the paper:
 *  (1) column-wise layout: the logits Z (B x V, as the model writes them) are transposed to
 *      Z^T (V x B) (each shard is transposed locally); here the transpose is fused
 *      with the penalty step;
 *  (2) incremental penalty buffers f in the same layout: dense per-(id, request) output
 *      counts and "seen" flags, updated in place for the B new tokens of every step (no rebuild);
 *      the penalty becomes one vectorised pass over Z^T;
 *  (3) memory reuse: the output buffer Y (L_max x B) is preallocated, new tokens appended as a row
 *      (P:370);
 *  vectorised (AVX-512: one vector = 16 requests at one vocabulary id) and multi-worker (pthreads,
 *  one group of 16 requests per worker at a time; the paper uses processes).
 * The sampling chain after the penalties follows the same definitions as the oracle and the GPU
 * path (R1-R12: OPENAI_CTRL penalties, temperature, softmax, top-k -> top-p over the
 * top-k -> min-p, inverse-CDF draw in ascending id with the Philox uniform keyed by (seed, request,
 * step)), in float32 values with float64 sums -- a production CPU sampler's precision, not the
 * oracle's.  Selection uses per-request histograms of M - z (1/32 nat bins), gathered/scattered
 * 16 requests at a time, so no per-request strided pass over the column-wise buffers is needed.
 */
#include <immintrin.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PC_LANES 16
#define PC_NB 1024      /* histogram bins of d = M - z: 1/32 nat each, the last one open-ended */
#define PC_BINS_PER 32.0f
#define PC_CCAP 16384   /* candidates kept per request (the exact top-k / cutoff-bin elements) */

typedef struct {
  float temperature, top_p, min_p, rep, pres, freq;
  int32_t top_k;
  uint64_t seed, request_id;
} pc_params;

typedef struct {
  int B, V, L, G, nthreads;   /* G groups of 16 requests */
  float* zt;                  /* [G][V][16] penalised, temperature-scaled logits of the step */
  float* cnt;                 /* [G][V][16] output-token counts (penalty buffer f) */
  uint8_t* seen;              /* [G][V][16] id in prompt or output (repetition penalty) */
  int32_t* Y;                 /* [L][B] output tokens */
  int32_t* nout;              /* [B] */
  pc_params* prm;             /* [B] */
  uint32_t* hc;               /* per worker: [PC_NB][16] histogram counts */
  double* hm;                 /*             [PC_NB][16] histogram masses */
  void* cbuf;                 /*             [16][PC_CCAP] candidates */
} pc_sampler;

/* ---------------------------------------------------------------- Philox4x32-10 (Salmon et al.) */
static double pc_uniform(uint64_t seed, uint64_t req, uint64_t step) {
  uint32_t c0 = (uint32_t)step, c1 = (uint32_t)(step >> 32), c2 = (uint32_t)req, c3 = (uint32_t)(req >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  const uint64_t x = ((uint64_t)c1 << 32) | c0;
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

/* ---------------------------------------------------------------- vector exp (x <= 0), ~2 ulp */
static inline __m512 pc_exp(__m512 x) {
  const __m512 l2e = _mm512_set1_ps(1.44269504088896341f);
  const __m512 ln2hi = _mm512_set1_ps(0.693359375f), ln2lo = _mm512_set1_ps(-2.12194440e-4f);
  x = _mm512_max_ps(x, _mm512_set1_ps(-100.0f));
  const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, l2e), _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  __m512 f = _mm512_fnmadd_ps(n, ln2hi, x);
  f = _mm512_fnmadd_ps(n, ln2lo, f);
  __m512 p = _mm512_set1_ps(1.0f / 720.0f);
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 120.0f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 24.0f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f / 6.0f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(0.5f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
  return _mm512_scalef_ps(p, n);
}

/* ---------------------------------------------------------------- handle */
pc_sampler* pc_create(int B, int V, int L, int nthreads) {
  pc_sampler* s = (pc_sampler*)calloc(1, sizeof(pc_sampler));
  if (!s) return NULL;
  s->B = B;
  s->V = V;
  s->L = L;
  s->G = (B + PC_LANES - 1) / PC_LANES;
  s->nthreads = nthreads < 1 ? 1 : nthreads;
  const size_t n = (size_t)s->G * V * PC_LANES;
  s->zt = (float*)aligned_alloc(64, n * sizeof(float));
  s->cnt = (float*)aligned_alloc(64, n * sizeof(float));
  s->seen = (uint8_t*)aligned_alloc(64, n);
  s->Y = (int32_t*)calloc((size_t)L * B, sizeof(int32_t));
  s->nout = (int32_t*)calloc(B, sizeof(int32_t));
  s->prm = (pc_params*)calloc(B, sizeof(pc_params));
  /* per-worker scratch allocated once (no page faults / allocator locks inside a step) */
  s->hc = (uint32_t*)aligned_alloc(64, sizeof(uint32_t) * PC_NB * PC_LANES * s->nthreads);
  s->hm = (double*)aligned_alloc(64, sizeof(double) * PC_NB * PC_LANES * s->nthreads);
  s->cbuf = aligned_alloc(64, 8 * (size_t)PC_CCAP * PC_LANES * s->nthreads);
  if (!s->zt || !s->cnt || !s->seen || !s->Y || !s->nout || !s->prm || !s->hc || !s->hm || !s->cbuf) return NULL;
  memset(s->hc, 0, sizeof(uint32_t) * PC_NB * PC_LANES * s->nthreads);
  memset(s->hm, 0, sizeof(double) * PC_NB * PC_LANES * s->nthreads);
  memset(s->cbuf, 0, 8 * (size_t)PC_CCAP * PC_LANES * s->nthreads);
  memset(s->cnt, 0, n * sizeof(float));
  memset(s->seen, 0, n);
  for (int b = 0; b < B; ++b) s->prm[b].temperature = 1.0f, s->prm[b].top_p = 1.0f, s->prm[b].rep = 1.0f;
  return s;
}

void pc_destroy(pc_sampler* s) {
  if (!s) return;
  free(s->zt);
  free(s->cnt);
  free(s->seen);
  free(s->Y);
  free(s->nout);
  free(s->prm);
  free(s->hc);
  free(s->hm);
  free(s->cbuf);
  free(s);
}

static inline size_t pc_at(const pc_sampler* s, int b, int v) {
  return ((size_t)(b / PC_LANES) * s->V + v) * PC_LANES + (b % PC_LANES);
}

void pc_set_params(pc_sampler* s, int b, float temperature, int32_t top_k, float top_p, float min_p, float rep,
                   float pres, float freq, uint64_t seed, uint64_t request_id) {
  pc_params p = {temperature, top_p, min_p, rep, pres, freq, top_k, seed, request_id};
  s->prm[b] = p;
}

/* the request's history: the penalty buffers rebuilt for this one column (admission) */
int pc_set_history(pc_sampler* s, int b, const int32_t* prompt, int np, const int32_t* out, int no) {
  if (no > s->L) return -1;
  for (int v = 0; v < s->V; ++v) {
    s->cnt[pc_at(s, b, v)] = 0.0f;
    s->seen[pc_at(s, b, v)] = 0;
  }
  for (int i = 0; i < np; ++i) s->seen[pc_at(s, b, prompt[i])] = 1;
  for (int i = 0; i < no; ++i) {
    s->cnt[pc_at(s, b, out[i])] += 1.0f;
    s->seen[pc_at(s, b, out[i])] = 1;
    s->Y[(size_t)i * s->B + b] = out[i];
  }
  s->nout[b] = no;
  return 0;
}

/* ---------------------------------------------------------------- one step */
typedef struct {
  pc_sampler* s;
  const void* logits;
  int is_bf16;
  int64_t ld;
  uint64_t step;
  int32_t* tokens;
  float* logprobs;
  int t, nt;
} pc_job;

typedef struct {
  float z;
  int32_t id;
} pc_cand;

static int pc_cmp_cand(const void* a, const void* b) {  /* z desc, id asc */
  const pc_cand* x = (const pc_cand*)a;
  const pc_cand* y = (const pc_cand*)b;
  if (x->z > y->z) return -1;
  if (x->z < y->z) return 1;
  return (x->id > y->id) - (x->id < y->id);
}

static int pc_cmp_id(const void* a, const void* b) {
  const pc_cand* x = (const pc_cand*)a;
  const pc_cand* y = (const pc_cand*)b;
  return (x->id > y->id) - (x->id < y->id);
}

static void pc_group(pc_sampler* s, int g, const pc_job* jb, uint32_t* hc, double* hm, pc_cand* cbuf, int ccap) {
  const int V = s->V, B = s->B;
  const int b0 = g * PC_LANES;
  float* zt = s->zt + (size_t)g * V * PC_LANES;
  const float* cnt = s->cnt + (size_t)g * V * PC_LANES;
  const uint8_t* seen = s->seen + (size_t)g * V * PC_LANES;
  float inv_tau[PC_LANES], rep[PC_LANES], pres[PC_LANES], freq[PC_LANES];
  int greedy[PC_LANES];
  for (int l = 0; l < PC_LANES; ++l) {
    const int b = b0 + l;
    const pc_params p = (b < B) ? s->prm[b] : s->prm[0];
    greedy[l] = p.temperature < 1e-5f;
    inv_tau[l] = greedy[l] ? 1.0f : 1.0f / p.temperature;
    rep[l] = p.rep;
    pres[l] = p.pres;
    freq[l] = p.freq;
  }
  const __m512 vinv = _mm512_loadu_ps(inv_tau), vrep = _mm512_loadu_ps(rep), vpres = _mm512_loadu_ps(pres),
               vfreq = _mm512_loadu_ps(freq), zero = _mm512_setzero_ps();
  /* pass 1: transpose 16 requests x 16 ids at a time, penalties (OPENAI_CTRL, R1) in
   * binary32, temperature; the running max */
  __m512 vmax = _mm512_set1_ps(-INFINITY);
  float tile[PC_LANES][PC_LANES];
  for (int v0 = 0; v0 < V; v0 += PC_LANES) {
    const int nv = (V - v0) < PC_LANES ? (V - v0) : PC_LANES;
    for (int l = 0; l < PC_LANES; ++l) {
      const int b = b0 + l < B ? b0 + l : B - 1;
      if (jb->is_bf16) {
        const uint16_t* row = (const uint16_t*)jb->logits + (size_t)b * jb->ld + v0;
        for (int j = 0; j < nv; ++j) {
          const uint32_t u = (uint32_t)row[j] << 16;
          memcpy(&tile[j][l], &u, 4);
        }
      } else {
        const float* row = (const float*)jb->logits + (size_t)b * jb->ld + v0;
        for (int j = 0; j < nv; ++j) tile[j][l] = row[j];
      }
    }
    for (int j = 0; j < nv; ++j) {
      const size_t o = (size_t)(v0 + j) * PC_LANES;
      __m512 x = _mm512_loadu_ps(tile[j]);
      const __m512 c = _mm512_load_ps(cnt + o);
      const __mmask16 sn = _mm512_test_epi32_mask(_mm512_cvtepu8_epi32(_mm_load_si128((const __m128i*)(seen + o))),
                                                  _mm512_set1_epi32(0xFF));
      /* y = y > 0 ? y / r : y * r for seen ids (r != 1); then y -= freq * cnt; y -= pres if cnt > 0 */
      const __m512 yr = _mm512_mask_blend_ps(_mm512_cmp_ps_mask(x, zero, _CMP_GT_OQ), _mm512_mul_ps(x, vrep),
                                             _mm512_div_ps(x, vrep));
      x = _mm512_mask_blend_ps(sn, x, yr);
      const __mmask16 hc_ = _mm512_cmp_ps_mask(c, zero, _CMP_GT_OQ);
      x = _mm512_mask_sub_ps(x, hc_, x, _mm512_mul_ps(vfreq, c));
      x = _mm512_mask_sub_ps(x, hc_, x, vpres);
      x = _mm512_mul_ps(x, vinv);
      _mm512_store_ps(zt + o, x);
      vmax = _mm512_max_ps(vmax, x);
    }
  }
  float M[PC_LANES];
  _mm512_storeu_ps(M, vmax);
  /* pass 2: S = sum exp(z - M) (float64 sums), histograms of d = M - z per request (count, mass),
   * the first id at the max (greedy) */
  memset(hc, 0, sizeof(uint32_t) * PC_NB * PC_LANES);
  memset(hm, 0, sizeof(double) * PC_NB * PC_LANES);
  __m512d s_lo = _mm512_setzero_pd(), s_hi = _mm512_setzero_pd();
  __m512i first = _mm512_set1_epi32(0x7FFFFFFF);
  const __m512i lane_off = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15);
  for (int v = 0; v < V; ++v) {
    const __m512 x = _mm512_load_ps(zt + (size_t)v * PC_LANES);
    const __mmask16 fin = _mm512_cmp_ps_mask(x, _mm512_set1_ps(-INFINITY), _CMP_GT_OQ);
    const __m512 d = _mm512_sub_ps(vmax, x);
    const __m512 w = _mm512_maskz_mov_ps(fin, pc_exp(_mm512_sub_ps(x, vmax)));
    s_lo = _mm512_add_pd(s_lo, _mm512_cvtps_pd(_mm512_castps512_ps256(w)));
    s_hi = _mm512_add_pd(s_hi, _mm512_cvtps_pd(_mm512_extractf32x8_ps(w, 1)));
    const __mmask16 atmax = _mm512_cmp_ps_mask(x, vmax, _CMP_EQ_OQ);
    first = _mm512_mask_min_epi32(first, atmax, first, _mm512_set1_epi32(v));
    __m512i bin = _mm512_cvttps_epi32(_mm512_min_ps(_mm512_mul_ps(d, _mm512_set1_ps(PC_BINS_PER)),
                                                    _mm512_set1_ps((float)(PC_NB - 1))));
    const __m512i idx = _mm512_add_epi32(_mm512_slli_epi32(bin, 4), lane_off);
    __m512i hcv = _mm512_mask_i32gather_epi32(_mm512_setzero_si512(), fin, idx, hc, 4);
    hcv = _mm512_add_epi32(hcv, _mm512_set1_epi32(1));
    _mm512_mask_i32scatter_epi32(hc, fin, idx, hcv, 4);
    const __m256i ilo = _mm512_castsi512_si256(idx), ihi = _mm512_extracti32x8_epi32(idx, 1);
    __m512d mlo = _mm512_mask_i32gather_pd(_mm512_setzero_pd(), (__mmask8)fin, ilo, hm, 8);
    __m512d mhi = _mm512_mask_i32gather_pd(_mm512_setzero_pd(), (__mmask8)(fin >> 8), ihi, hm, 8);
    mlo = _mm512_add_pd(mlo, _mm512_cvtps_pd(_mm512_castps512_ps256(w)));
    mhi = _mm512_add_pd(mhi, _mm512_cvtps_pd(_mm512_extractf32x8_ps(w, 1)));
    _mm512_mask_i32scatter_pd(hm, (__mmask8)fin, ilo, mlo, 8);
    _mm512_mask_i32scatter_pd(hm, (__mmask8)(fin >> 8), ihi, mhi, 8);
  }
  double S[PC_LANES];
  _mm512_storeu_pd(S, s_lo);
  _mm512_storeu_pd(S + 8, s_hi);
  int32_t firstm[PC_LANES];
  _mm512_storeu_si512(firstm, first);
  /* per request: the cutoff bin from the histograms, then the exact cutoff among that bin's (or the
   * top-k bins') elements; the kept set K3 = {z > zc} + {z == zc, id <= idc} (+ min-p) */
  float zc[PC_LANES], zmin[PC_LANES];
  int32_t idc[PC_LANES], cbin[PC_LANES];
  double Wk[PC_LANES], tgt[PC_LANES];
  int bounded[PC_LANES], nk[PC_LANES];
  pc_cand* kept[PC_LANES];
  int need_pass = 0;
  for (int l = 0; l < PC_LANES; ++l) {
    kept[l] = NULL;
    nk[l] = 0;
    bounded[l] = 0;
    zc[l] = -INFINITY;
    idc[l] = 0x7FFFFFFF;
    cbin[l] = PC_NB - 1;
    zmin[l] = -INFINITY;
    Wk[l] = 0.0;
    const int b = b0 + l;
    if (b >= B || greedy[l] || !(M[l] > -INFINITY)) continue;
    const pc_params p = s->prm[b];
    if (p.min_p > 0.0f) zmin[l] = logf(p.min_p);  /* w >= min_p  <=>  z - M >= ln(min_p) */
    if (p.top_k >= 1 && p.top_k < V) {
      uint32_t c = 0;
      int kb = PC_NB - 1;
      for (int i = 0; i < PC_NB; ++i) {
        c += hc[i * PC_LANES + l];
        if (c >= (uint32_t)p.top_k) {
          kb = i;
          break;
        }
      }
      cbin[l] = kb;
      bounded[l] = 1;
    } else if (p.top_p < 1.0f) {
      const double target = (double)p.top_p * S[l];
      double m = 0.0;
      int pb = PC_NB - 1;
      for (int i = 0; i < PC_NB; ++i) {
        if (m + hm[i * PC_LANES + l] >= target) {
          pb = i;
          break;
        }
        m += hm[i * PC_LANES + l];
      }
      cbin[l] = pb;
      Wk[l] = m;  /* mass of the bins before the cutoff bin */
      bounded[l] = 0;
    } else {
      cbin[l] = -1;  /* no cutoff: everything finite (min-p aside) is kept */
    }
    need_pass = 1;
  }
  /* pass 3: the elements of each request's candidate bins (bounded: bins <= cbin; top-p: == cbin) */
  int ncand[PC_LANES] = {0};
  if (need_pass) {
    int32_t cb[PC_LANES], bd[PC_LANES];
    for (int l = 0; l < PC_LANES; ++l) cb[l] = cbin[l], bd[l] = bounded[l];
    const __m512i vcb = _mm512_loadu_si512(cb), vbd = _mm512_loadu_si512(bd);
    const __mmask16 isb = _mm512_test_epi32_mask(vbd, vbd);
    for (int v = 0; v < V; ++v) {
      const __m512 x = _mm512_load_ps(zt + (size_t)v * PC_LANES);
      const __m512i bin = _mm512_cvttps_epi32(_mm512_min_ps(_mm512_mul_ps(_mm512_sub_ps(vmax, x), _mm512_set1_ps(PC_BINS_PER)),
                                                            _mm512_set1_ps((float)(PC_NB - 1))));
      const __mmask16 fin = _mm512_cmp_ps_mask(x, _mm512_set1_ps(-INFINITY), _CMP_GT_OQ);
      __mmask16 hit = (isb & _mm512_cmple_epi32_mask(bin, vcb)) | (~isb & _mm512_cmpeq_epi32_mask(bin, vcb));
      hit &= fin;
      while (hit) {
        const int l = __builtin_ctz(hit);
        hit &= hit - 1;
        if (ncand[l] < ccap) {
          cbuf[(size_t)l * ccap + ncand[l]].z = zt[(size_t)v * PC_LANES + l];
          cbuf[(size_t)l * ccap + ncand[l]].id = v;
        }
        ++ncand[l];
      }
    }
  }
  for (int l = 0; l < PC_LANES; ++l) {
    const int b = b0 + l;
    if (b >= B) continue;
    const pc_params p = s->prm[b];
    const double u = pc_uniform(p.seed, p.request_id, jb->step);
    if (!(M[l] > -INFINITY)) {
      jb->tokens[b] = -1;
      jb->logprobs[b] = NAN;
      continue;
    }
    if (greedy[l]) {
      jb->tokens[b] = firstm[l];
      jb->logprobs[b] = (float)(-log(S[l]));
      continue;
    }
    pc_cand* cl = cbuf + (size_t)l * ccap;
    const int n = ncand[l] < ccap ? ncand[l] : ccap;
    if (cbin[l] >= 0) qsort(cl, n, sizeof(pc_cand), pc_cmp_cand);
    /* the kept prefix of the candidates (pi order) */
    int nkeep = 0;
    double W = 0.0;
    if (bounded[l]) {
      int k1 = p.top_k < n ? p.top_k : n;
      double W1 = 0.0;
      for (int i = 0; i < k1; ++i) W1 += exp((double)(cl[i].z - M[l]));
      int k2 = k1;
      if (p.top_p < 1.0f) {
        const double target = (double)p.top_p * W1;
        double c = 0.0;
        for (int i = 0; i < k1; ++i) {
          c += exp((double)(cl[i].z - M[l]));
          if (c >= target) {
            k2 = i + 1;
            break;
          }
        }
      }
      int k3 = 0;
      for (int i = 0; i < k2; ++i)
        if (cl[i].z - M[l] >= zmin[l]) cl[k3++] = cl[i];
      nkeep = k3;
      for (int i = 0; i < nkeep; ++i) W += exp((double)(cl[i].z - M[l]));
      zc[l] = nkeep ? cl[nkeep - 1].z : INFINITY;
      idc[l] = nkeep ? cl[nkeep - 1].id : -1;
      /* bounded: the draw over the (small) kept set in id order */
      qsort(cl, nkeep, sizeof(pc_cand), pc_cmp_id);
      const double target = u * W;
      double c = 0.0;
      int tok = nkeep ? cl[nkeep - 1].id : -1;
      float ztok = nkeep ? cl[nkeep - 1].z : NAN;
      for (int i = 0; i < nkeep; ++i) {
        c += exp((double)(cl[i].z - M[l]));
        if (c > target) {
          tok = cl[i].id;
          ztok = cl[i].z;
          break;
        }
      }
      jb->tokens[b] = tok;
      jb->logprobs[b] = (float)((double)(ztok - M[l]) - log(S[l]));
      nk[l] = -1;  /* done */
    } else if (cbin[l] >= 0) {
      /* top-p without top-k: the cutoff inside bin cbin by its sorted elements */
      const double target = (double)p.top_p * S[l];
      double c = Wk[l];
      int j = n - 1;
      for (int i = 0; i < n; ++i) {
        c += exp((double)(cl[i].z - M[l]));
        if (c >= target) {
          j = i;
          break;
        }
      }
      zc[l] = n ? cl[j].z : INFINITY;
      idc[l] = n ? cl[j].id : -1;
      nk[l] = 0;
    } else {
      zc[l] = -INFINITY;
      idc[l] = 0x7FFFFFFF;
      nk[l] = 0;
    }
  }
  /* pass 4 (unbounded requests): W over K3, then the first id whose cumulative kept mass > u W */
  int anyu = 0;
  for (int l = 0; l < PC_LANES; ++l)
    if (b0 + l < B && nk[l] == 0 && !greedy[l] && M[l] > -INFINITY) anyu = 1;
  if (anyu) {
    __mmask16 act = 0;
    for (int l = 0; l < PC_LANES; ++l)
      if (b0 + l < B && nk[l] == 0 && !greedy[l] && M[l] > -INFINITY) act |= (__mmask16)(1u << l);
    float zcl[PC_LANES], zml[PC_LANES];
    int32_t idl[PC_LANES];
    for (int l = 0; l < PC_LANES; ++l) zcl[l] = zc[l], idl[l] = idc[l], zml[l] = zmin[l];
    const __m512 vzc = _mm512_loadu_ps(zcl), vzm = _mm512_loadu_ps(zml);
    const __m512i vid = _mm512_loadu_si512(idl);
    /* W in id order (float64, 8 + 8 lanes) */
    __m512d w_lo = _mm512_setzero_pd(), w_hi = _mm512_setzero_pd();
    for (int v = 0; v < V; ++v) {
      const __m512 x = _mm512_load_ps(zt + (size_t)v * PC_LANES);
      const __mmask16 k = act & (_mm512_cmp_ps_mask(x, vzc, _CMP_GT_OQ) |
                                 (_mm512_cmp_ps_mask(x, vzc, _CMP_EQ_OQ) & _mm512_cmple_epi32_mask(_mm512_set1_epi32(v), vid))) &
                          _mm512_cmp_ps_mask(_mm512_sub_ps(x, vmax), vzm, _CMP_GE_OQ);
      const __m512 w = _mm512_maskz_mov_ps(k, pc_exp(_mm512_sub_ps(x, vmax)));
      w_lo = _mm512_add_pd(w_lo, _mm512_cvtps_pd(_mm512_castps512_ps256(w)));
      w_hi = _mm512_add_pd(w_hi, _mm512_cvtps_pd(_mm512_extractf32x8_ps(w, 1)));
    }
    double Wl[PC_LANES], T[PC_LANES];
    _mm512_storeu_pd(Wl, w_lo);
    _mm512_storeu_pd(Wl + 8, w_hi);
    for (int l = 0; l < PC_LANES; ++l) {
      const int b = b0 + l;
      T[l] = (b < B) ? pc_uniform(s->prm[b].seed, s->prm[b].request_id, jb->step) * Wl[l] : 0.0;
      tgt[l] = T[l];
    }
    const __m512d t_lo = _mm512_loadu_pd(T), t_hi = _mm512_loadu_pd(T + 8);
    __m512d c_lo = _mm512_setzero_pd(), c_hi = _mm512_setzero_pd();
    __m512i pick = _mm512_set1_epi32(-1), lastk = _mm512_set1_epi32(-1);
    __mmask16 open = act;
    for (int v = 0; v < V && open; ++v) {
      const __m512 x = _mm512_load_ps(zt + (size_t)v * PC_LANES);
      const __mmask16 k = open & (_mm512_cmp_ps_mask(x, vzc, _CMP_GT_OQ) |
                                  (_mm512_cmp_ps_mask(x, vzc, _CMP_EQ_OQ) & _mm512_cmple_epi32_mask(_mm512_set1_epi32(v), vid))) &
                          _mm512_cmp_ps_mask(_mm512_sub_ps(x, vmax), vzm, _CMP_GE_OQ);
      if (!k) continue;
      const __m512 w = _mm512_maskz_mov_ps(k, pc_exp(_mm512_sub_ps(x, vmax)));
      c_lo = _mm512_add_pd(c_lo, _mm512_cvtps_pd(_mm512_castps512_ps256(w)));
      c_hi = _mm512_add_pd(c_hi, _mm512_cvtps_pd(_mm512_extractf32x8_ps(w, 1)));
      lastk = _mm512_mask_mov_epi32(lastk, k, _mm512_set1_epi32(v));
      const __mmask16 cross = k & (__mmask16)(_mm512_cmp_pd_mask(c_lo, t_lo, _CMP_GT_OQ) |
                                              ((__mmask16)_mm512_cmp_pd_mask(c_hi, t_hi, _CMP_GT_OQ) << 8));
      pick = _mm512_mask_mov_epi32(pick, cross, _mm512_set1_epi32(v));
      open &= ~cross;
    }
    int32_t pk[PC_LANES], lk[PC_LANES];
    _mm512_storeu_si512(pk, pick);
    _mm512_storeu_si512(lk, lastk);
    for (int l = 0; l < PC_LANES; ++l) {
      if (!((act >> l) & 1)) continue;
      const int b = b0 + l;
      const int tok = pk[l] >= 0 ? pk[l] : lk[l];
      jb->tokens[b] = tok;
      jb->logprobs[b] = tok >= 0 ? (float)((double)(zt[(size_t)tok * PC_LANES + l] - M[l]) - log(S[l])) : NAN;
    }
  }
}

static void* pc_worker(void* arg) {
  pc_job* jb = (pc_job*)arg;
  pc_sampler* s = jb->s;
  uint32_t* hc = s->hc + (size_t)jb->t * PC_NB * PC_LANES;
  double* hm = s->hm + (size_t)jb->t * PC_NB * PC_LANES;
  pc_cand* cbuf = (pc_cand*)s->cbuf + (size_t)jb->t * PC_CCAP * PC_LANES;
  for (int g = jb->t; g < s->G; g += jb->nt) pc_group(s, g, jb, hc, hm, cbuf, PC_CCAP);
  return NULL;
}

/* One sampling step for all B requests: logits [B x ld] (bf16 bit patterns or float32), tokens and
 * logprobs out; then the incremental update of the penalty buffers and Y with the B new tokens. */
int pc_step(pc_sampler* s, const void* logits, int is_bf16, int64_t ld, uint64_t step, int32_t* tokens, float* logprobs,
            int append) {
  const int nt = s->nthreads < s->G ? s->nthreads : s->G;
  pthread_t th[256];
  pc_job jobs[256];
  for (int t = 0; t < nt; ++t) {
    pc_job j = {s, logits, is_bf16, ld, step, tokens, logprobs, t, nt};
    jobs[t] = j;
    if (t) pthread_create(&th[t], NULL, pc_worker, &jobs[t]);
  }
  pc_worker(&jobs[0]);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
  if (append) {  /* only the B entries of the new tokens change */
    for (int b = 0; b < s->B; ++b) {
      const int tok = tokens[b];
      if (tok < 0 || s->nout[b] >= s->L) continue;
      s->cnt[pc_at(s, b, tok)] += 1.0f;
      s->seen[pc_at(s, b, tok)] = 1;
      s->Y[(size_t)s->nout[b] * s->B + b] = tok;
      s->nout[b] += 1;
    }
  }
  return 0;
}

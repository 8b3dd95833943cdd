// sampler.cu — C-ABI implementation (host side) of include/sampler.h.
//
// Owns per-handle device state (params table, per-slot history + incremental unique-token
// penalty table, workspace), validates every call on the host before any launch, and enqueues
// the sm_100a kernels on the caller's stream: phase A (stream.cuh), phase B (select.cuh, launched
// with programmatic dependent launch so its prologue overlaps phase A's tail), the exact
// multi-pass kernel (exact.cuh) only when some row can stay unresolved, and the sharded merge
// (merge.cuh).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "exact.cuh"
#include "merge.cuh"
#include "resolve.cuh"
#include "select.cuh"
#include "stream.cuh"

using namespace smp;

struct sampler {
  sampler_config cfg{};
  int sm_count = 0;
  int Vp = 0;    // vocab_local rounded up to the vector width
  int vec = 8;   // elements per 16 bytes
  int64_t Vq = 0;  // padded row length in vectors (piece.cuh)
  int max_ctas = 0;
  int64_t rec_stride = 0;
  // device state
  sampling_params* d_params = nullptr;
  SlotMeta* d_meta = nullptr;
  UniqEntry* d_uniq = nullptr;
  int32_t* d_hist = nullptr;
  RowInfo* d_info = nullptr;
  ResState* d_rs = nullptr;     // [max_batch] NEXT-1 resolve rounds (resolve.cuh)
  const uint64_t* d_step_src = nullptr;  // sampler_set_step_source: the decode step read on the device
  // NEXT-2 one-shot peer exchange (common.cuh ExchPeers)
  uint8_t* d_xbuf = nullptr;     // this rank's exchange buffer (records x 2 parities + flags)
  uint8_t** d_xbases = nullptr;  // [world] device copy of every rank's mapped base
  uint32_t* d_xseq = nullptr;    // [3][max_batch] publish / merge / resolve sequence numbers
  std::vector<void*> x_opened;   // IPC mappings to close
  int x_world = 0, x_rank = 0;
  int64_t x_bytes = 0;
  int64_t x_res_off = 0;         // the resolve payload region inside the exchange buffer
  uint64_t x_timeout_ns = 0;
  uint32_t* d_pmask = nullptr;  // [max_batch][spr * 32] penalty presence bitmaps (HistState)
  PartRec* d_parts = nullptr;   // [max_batch][rpr_max][kCW] phase-A partial records
  RowHand* d_hand = nullptr;    // [max_batch] phase A -> B hand-off
  PenEnt* d_pent = nullptr;     // [max_batch][max_history] penalised entries (hand-off)
  uint16_t* d_gkeys = nullptr;  // [max_batch][Vq/4] group keys (phase A -> phase B)
  uint64_t* d_trace = nullptr;
  // host mirror
  std::vector<sampling_params> h_params;
  std::string err;
  int32_t last_launches = 0;
  // per-kernel timing (sampler_set_timing)
  bool timing = false;
  cudaEvent_t tev[4] = {};
  int tev_n = 0;  // kernels timed by the last call
};

// event after the k-th kernel of a call (k = 0: before the first)
static void tmark(sampler* h, int k, cudaStream_t st) {
  if (!h->timing) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  // under graph capture the marks must be external event nodes to be readable after a replay
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(h->tev[k], st, cudaEventRecordExternal);
  else cudaEventRecord(h->tev[k], st);
  h->tev_n = k;
}

static HistState hist_state(const sampler* h) {
  HistState s;
  s.meta = h->d_meta;
  s.uniq = h->d_uniq;
  s.tokens = h->d_hist;
  s.L = h->cfg.max_history;
  s.nslots = h->cfg.max_batch;
  s.pmask = h->d_pmask;
  s.spr = (int)(h->Vq / kStepVec);
  s.vec = h->vec;
  s.voff = h->cfg.vocab_offset;
  s.vloc = h->cfg.vocab_local;
  return s;
}

static int64_t trace_a_len(const sampler* h) {  // phase-A trace entries (64 per CTA, worst-case grid)
  return 64 * ((int64_t)h->cfg.max_batch * (h->Vq / kStepVec) / kTileSteps + 1);
}

static thread_local std::string g_create_err;

static int fail(sampler* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h)
    h->err = buf;
  else
    g_create_err = buf;
  return code;
}

#define CK(h, call)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail((h), SAMPLER_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
  } while (0)

static const char* param_error(const sampling_params& p, int pen_mode) {
  if (!(p.temperature >= 0.0f) || !std::isfinite(p.temperature)) return "temperature must be finite and >= 0";
  if (!(p.top_p > 0.0f && p.top_p <= 1.0f)) return "top_p must be in (0, 1]";
  if (!(p.min_p >= 0.0f && p.min_p <= 1.0f)) return "min_p must be in [0, 1]";
  if (!std::isfinite(p.repetition_penalty) || !std::isfinite(p.presence_penalty) ||
      !std::isfinite(p.frequency_penalty))
    return "penalties must be finite";
  if (pen_mode == SAMPLER_PEN_OPENAI_CTRL && !(p.repetition_penalty > 0.0f))
    return "repetition_penalty must be > 0 (OPENAI_CTRL mode)";
  if (p.reserved != 0) return "reserved must be 0";
  return nullptr;
}

static bool row_may_pend(const sampling_params& p, int V, int kcand) {
  if (p.temperature < kGreedyEps) return false;
  if (p.top_k >= 1 && p.top_k < V && p.top_k <= kcand) return false;
  return true;
}

extern "C" {

const char* sampler_version(void) {
  return "paper_2506_22033_b200 sampler: sm_100a (compute_100a); phase A: persistent warp-specialised "
         "stream (1-D bulk-copy ring, penalty presence bitmap, packed bf16 exp-sum, group/step keys); "
         "phase B: per-row step-key bound, group re-read, exact top-k, candidate-parallel decision, "
         "Philox4x32-10; exact float64 cluster kernel for unbounded rows; vocab-sharded: NCCL or one-shot "
         "peer exchange (fused merge), distributed resolve rounds";
}

const char* sampler_last_error(const sampler* h) { return h ? h->err.c_str() : g_create_err.c_str(); }

int32_t sampler_last_launch_count(const sampler* h) { return h ? h->last_launches : 0; }

int sampler_set_timing(sampler* h, int32_t enable) {
  if (!h) return SAMPLER_EINVAL;
  cudaSetDevice(h->cfg.device);
  if (enable && !h->tev[0])
    for (auto& e : h->tev) CK(h, cudaEventCreate(&e));
  h->timing = enable != 0;
  h->tev_n = 0;
  return SAMPLER_OK;
}

int sampler_kernel_times(sampler* h, float* ms_out, int32_t n, int32_t* count) {
  if (!h || !ms_out || !count) return SAMPLER_EINVAL;
  if (!h->timing || h->tev_n < 1) return fail(h, SAMPLER_EINVAL, "timing off or nothing timed");
  CK(h, cudaEventSynchronize(h->tev[h->tev_n]));
  for (int k = 0; k < h->tev_n && k < n; ++k) CK(h, cudaEventElapsedTime(&ms_out[k], h->tev[k], h->tev[k + 1]));
  *count = h->tev_n;
  return SAMPLER_OK;
}

int sampler_create(const sampler_config* cfg, sampler** out) {
  if (!out) return fail(nullptr, SAMPLER_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, SAMPLER_EINVAL, "cfg is NULL");
  const sampler_config c = *cfg;
  if (c.vocab_size < 1 || c.vocab_size > (int32_t)(0x7FFFFFFF - (1 << 20)))
    return fail(nullptr, SAMPLER_EINVAL, "vocab_size out of range");
  if (c.vocab_offset < 0 || c.vocab_local < 1 || (int64_t)c.vocab_offset + c.vocab_local > c.vocab_size)
    return fail(nullptr, SAMPLER_EINVAL, "vocab slice out of range");
  if (c.max_batch < 1 || c.max_batch > (1 << 20)) return fail(nullptr, SAMPLER_EINVAL, "max_batch out of range");
  if (c.max_history < 1 || c.max_history > (1 << 24))
    return fail(nullptr, SAMPLER_EINVAL, "max_history out of range");
  if (c.max_top_k < 1 || c.max_top_k > SAMPLER_KCAND_MAX)
    return fail(nullptr, SAMPLER_EINVAL, "max_top_k must be in [1, %d]", SAMPLER_KCAND_MAX);
  if (c.logits_dtype != SAMPLER_F32 && c.logits_dtype != SAMPLER_BF16)
    return fail(nullptr, SAMPLER_EUNSUPPORTED, "logits_dtype must be SAMPLER_F32 or SAMPLER_BF16");
  if (c.penalty_mode != SAMPLER_PEN_OPENAI_CTRL && c.penalty_mode != SAMPLER_PEN_LINEAR)
    return fail(nullptr, SAMPLER_EINVAL, "bad penalty_mode");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
    return fail(nullptr, SAMPLER_ECUDA, "no CUDA device");
  if (c.device < 0 || c.device >= ndev) return fail(nullptr, SAMPLER_EINVAL, "bad device ordinal");
  if (cudaSetDevice(c.device) != cudaSuccess) return fail(nullptr, SAMPLER_ECUDA, "cudaSetDevice failed");

  sampler* h = new sampler();
  h->cfg = c;
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, c.device);
  h->vec = (c.logits_dtype == SAMPLER_BF16) ? 8 : 4;
  h->Vp = (c.vocab_local + h->vec - 1) / h->vec * h->vec;
  h->max_ctas = h->sm_count;
  h->Vq = vq_of(c.vocab_local, h->vec);
  h->rec_stride = (rec_stride_bytes(c.max_top_k) + 127) / 128 * 128;
  const int64_t B = c.max_batch, L = c.max_history;
  auto al = [&](void** p, size_t n) -> bool { return cudaMalloc(p, n) == cudaSuccess; };
  bool ok = al((void**)&h->d_params, sizeof(sampling_params) * B) &&
            al((void**)&h->d_meta, sizeof(SlotMeta) * B) && al((void**)&h->d_uniq, sizeof(UniqEntry) * (B * L + 4))  /* (+4: phase A's 16-byte bulk copies) */ &&
            al((void**)&h->d_hist, sizeof(int32_t) * B * L) && al((void**)&h->d_info, sizeof(RowInfo) * B) &&
            al((void**)&h->d_rs, sizeof(ResState) * B) &&
            al((void**)&h->d_gkeys, sizeof(uint16_t) * B * gk_stride(h->Vq)) &&
            al((void**)&h->d_pmask, sizeof(uint32_t) * B * (h->Vq / kStepVec) * 32) &&
            al((void**)&h->d_hand, sizeof(RowHand) * B) &&  al((void**)&h->d_pent, sizeof(PenEnt) * B * L) &&
            al((void**)&h->d_parts, sizeof(PartRec) * B * kCW * ((h->Vq / kStepVec + kTileSteps - 1) / kTileSteps + 1));
  if (!ok) {
    cudaGetLastError();
    sampler_destroy(h);
    return fail(nullptr, SAMPLER_ENOMEM, "device allocation failed");
  }
  h->h_params.resize(B);
  for (int64_t i = 0; i < B; ++i) {
    sampling_params p{};
    p.temperature = 1.0f;
    p.top_k = 0;
    p.top_p = 1.0f;
    p.min_p = 0.0f;
    p.repetition_penalty = (c.penalty_mode == SAMPLER_PEN_LINEAR) ? 0.0f : 1.0f;
    p.presence_penalty = 0.0f;
    p.frequency_penalty = 0.0f;
    p.reserved = 0;
    p.seed = 0;
    p.request_id = (uint64_t)i;
    h->h_params[i] = p;
  }
  if (cudaMemcpy(h->d_params, h->h_params.data(), sizeof(sampling_params) * B, cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cudaMemset(h->d_meta, 0, sizeof(SlotMeta) * B) != cudaSuccess ||
      cudaMemset(h->d_pmask, 0, sizeof(uint32_t) * B * (h->Vq / kStepVec) * 32) != cudaSuccess ||
      cudaMemset(h->d_info, 0, sizeof(RowInfo) * B) != cudaSuccess ||
      cudaMemset(h->d_rs, 0, sizeof(ResState) * B) != cudaSuccess ||
      cudaFuncSetAttribute(stream_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kStreamSmem) != cudaSuccess ||
      cudaFuncSetAttribute(stream_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem) !=
          cudaSuccess ||
      cudaFuncSetAttribute(exact_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kExactSmemBf16) != cudaSuccess ||
      cudaFuncSetAttribute(select_rows_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kSelectSmem) != cudaSuccess ||
      cudaFuncSetAttribute(select_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelectSmem) !=
          cudaSuccess ||
      cudaFuncSetAttribute(exact_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExactSmem) !=
          cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    const char* m = cudaGetErrorString(cudaGetLastError());
    sampler_destroy(h);
    return fail(nullptr, SAMPLER_ECUDA, "device init failed: %s", m);
  }
#ifdef SMP_CARVEOUT
  // one L1/shared split for every kernel of the step: no reconfiguration at the kernel boundaries
  cudaFuncSetAttribute(stream_kernel<__nv_bfloat16>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
  cudaFuncSetAttribute(stream_kernel<float>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
  cudaFuncSetAttribute(select_rows_kernel<__nv_bfloat16>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
  cudaFuncSetAttribute(select_rows_kernel<float>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
  cudaFuncSetAttribute(exact_kernel<__nv_bfloat16>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
  cudaFuncSetAttribute(exact_kernel<float>, cudaFuncAttributePreferredSharedMemoryCarveout, SMP_CARVEOUT);
#endif
  if (getenv("SAMPLER_TRACE")) {
    if (cudaMalloc((void**)&h->d_trace, sizeof(uint64_t) * (trace_a_len(h) + 32 * (int64_t)B)) != cudaSuccess) h->d_trace = nullptr;
  }
  *out = h;
  return SAMPLER_OK;
}

int sampler_destroy(sampler* h) {
  if (!h) return SAMPLER_OK;
  cudaSetDevice(h->cfg.device);
  cudaFree(h->d_params);
  cudaFree(h->d_meta);
  cudaFree(h->d_uniq);
  cudaFree(h->d_hist);
  cudaFree(h->d_info);
  cudaFree(h->d_rs);
  for (void* p : h->x_opened) cudaIpcCloseMemHandle(p);
  cudaFree(h->d_xbuf);
  cudaFree(h->d_xbases);
  cudaFree(h->d_xseq);
  cudaFree(h->d_trace);
  cudaFree(h->d_gkeys);
  cudaFree(h->d_pmask);
  cudaFree(h->d_parts);
  cudaFree(h->d_hand);
  cudaFree(h->d_pent);
  for (auto& e : h->tev)
    if (e) cudaEventDestroy(e);
  delete h;
  return SAMPLER_OK;
}

int sampler_set_params(sampler* h, int32_t n, const int32_t* slots, const sampling_params* params) {
  if (!h) return SAMPLER_EINVAL;
  if (n < 0 || (n > 0 && (!slots || !params))) return fail(h, SAMPLER_EINVAL, "bad arguments");
  for (int32_t i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= h->cfg.max_batch) return fail(h, SAMPLER_ERANGE, "slot %d out of range", slots[i]);
    const char* e = param_error(params[i], h->cfg.penalty_mode);
    if (e) return fail(h, SAMPLER_EINVAL, "params[%d]: %s", i, e);
  }
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaDeviceSynchronize());  // no in-flight sample may still read the table (sampler.h)
  for (int32_t i = 0; i < n; ++i) {
    h->h_params[slots[i]] = params[i];
    CK(h, cudaMemcpy(h->d_params + slots[i], &params[i], sizeof(sampling_params), cudaMemcpyHostToDevice));
  }
  return SAMPLER_OK;
}

static int upload_slot(sampler* h, int slot, const std::vector<int32_t>& prompt, const std::vector<int32_t>& output,
                       int32_t flags) {
  const int L = h->cfg.max_history;
  std::map<int32_t, uint32_t> m;
  for (int32_t t : prompt) m[t] |= 1u;
  for (int32_t t : output) m[t] += 2u;
  std::vector<UniqEntry> u;
  u.reserve(m.size());
  for (auto& kv : m) {
    UniqEntry e;
    e.id = kv.first;
    e.meta = kv.second;
    u.push_back(e);
  }
  std::vector<int32_t> toks(prompt);
  toks.insert(toks.end(), output.begin(), output.end());
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaDeviceSynchronize());  // no in-flight sample may still append to this slot (sampler.h)
  SlotMeta sm;
  sm.n_prompt = (int32_t)prompt.size();
  sm.n_out = (int32_t)output.size();
  sm.n_uniq = (int32_t)u.size();
  sm.flags = flags;
  CK(h, cudaSetDevice(h->cfg.device));
  if (!u.empty())
    CK(h, cudaMemcpy(h->d_uniq + (int64_t)slot * L, u.data(), sizeof(UniqEntry) * u.size(), cudaMemcpyHostToDevice));
  if (!toks.empty())
    CK(h, cudaMemcpy(h->d_hist + (int64_t)slot * L, toks.data(), sizeof(int32_t) * toks.size(), cudaMemcpyHostToDevice));
  // penalty presence bitmap of the slot (HistState::pmask)
  const int64_t nw = (h->Vq / kStepVec) * 32;
  std::vector<uint32_t> pm(nw, 0u);
  for (const UniqEntry& e : u) {
    const int le = e.id - h->cfg.vocab_offset;
    if (le < 0 || le >= h->cfg.vocab_local) continue;
    int w;
    uint32_t b;
    pmask_pos(le, h->vec, &w, &b);
    pm[w] |= b;
  }
  CK(h, cudaMemcpy(h->d_pmask + (int64_t)slot * nw, pm.data(), sizeof(uint32_t) * nw, cudaMemcpyHostToDevice));
  CK(h, cudaMemcpy(h->d_meta + slot, &sm, sizeof(SlotMeta), cudaMemcpyHostToDevice));
  return SAMPLER_OK;
}

int sampler_set_history(sampler* h, int32_t slot, const int32_t* prompt, int32_t n_prompt, const int32_t* output,
                        int32_t n_output) {
  if (!h) return SAMPLER_EINVAL;
  if (slot < 0 || slot >= h->cfg.max_batch) return fail(h, SAMPLER_ERANGE, "slot %d out of range", slot);
  if (n_prompt < 0 || n_output < 0 || (n_prompt > 0 && !prompt) || (n_output > 0 && !output))
    return fail(h, SAMPLER_EINVAL, "bad history arguments");
  if ((int64_t)n_prompt + n_output > h->cfg.max_history)
    return fail(h, SAMPLER_ERANGE, "history %d exceeds max_history %d", n_prompt + n_output, h->cfg.max_history);
  for (int32_t i = 0; i < n_prompt; ++i)
    if (prompt[i] < 0 || prompt[i] >= h->cfg.vocab_size) return fail(h, SAMPLER_ERANGE, "prompt token out of range");
  for (int32_t i = 0; i < n_output; ++i)
    if (output[i] < 0 || output[i] >= h->cfg.vocab_size) return fail(h, SAMPLER_ERANGE, "output token out of range");
  std::vector<int32_t> p(prompt, prompt + n_prompt), o(output, output + n_output);
  return upload_slot(h, slot, p, o, 0);
}

static int read_slot(sampler* h, int slot, SlotMeta* sm, std::vector<int32_t>* toks, std::vector<UniqEntry>* u) {
  const int L = h->cfg.max_history;
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaMemcpy(sm, h->d_meta + slot, sizeof(SlotMeta), cudaMemcpyDeviceToHost));
  if (toks) {
    toks->resize(sm->n_prompt + sm->n_out);
    if (!toks->empty())
      CK(h, cudaMemcpy(toks->data(), h->d_hist + (int64_t)slot * L, sizeof(int32_t) * toks->size(),
                       cudaMemcpyDeviceToHost));
  }
  if (u) {
    u->resize(sm->n_uniq);
    if (!u->empty())
      CK(h, cudaMemcpy(u->data(), h->d_uniq + (int64_t)slot * L, sizeof(UniqEntry) * u->size(),
                       cudaMemcpyDeviceToHost));
  }
  return SAMPLER_OK;
}

int sampler_append_tokens(sampler* h, int32_t n, const int32_t* slots, const int32_t* tokens) {
  if (!h) return SAMPLER_EINVAL;
  if (n < 0 || (n > 0 && (!slots || !tokens))) return fail(h, SAMPLER_EINVAL, "bad arguments");
  std::vector<SlotMeta> metas(n);
  for (int32_t i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= h->cfg.max_batch) return fail(h, SAMPLER_ERANGE, "slot out of range");
    if (tokens[i] < 0 || tokens[i] >= h->cfg.vocab_size) return fail(h, SAMPLER_ERANGE, "token out of range");
  }
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaDeviceSynchronize());
  // capacity check for all first (per slot, counting repeats within this call)
  std::map<int32_t, int> add;
  for (int32_t i = 0; i < n; ++i) add[slots[i]]++;
  for (auto& kv : add) {
    SlotMeta sm;
    CK(h, cudaMemcpy(&sm, h->d_meta + kv.first, sizeof(SlotMeta), cudaMemcpyDeviceToHost));
    if ((int64_t)sm.n_prompt + sm.n_out + kv.second > h->cfg.max_history)
      return fail(h, SAMPLER_ERANGE, "slot %d would exceed max_history", kv.first);
  }
  for (int32_t i = 0; i < n; ++i) {
    SlotMeta sm;
    std::vector<int32_t> toks;
    int rc = read_slot(h, slots[i], &sm, &toks, nullptr);
    if (rc) return rc;
    std::vector<int32_t> p(toks.begin(), toks.begin() + sm.n_prompt), o(toks.begin() + sm.n_prompt, toks.end());
    o.push_back(tokens[i]);
    rc = upload_slot(h, slots[i], p, o, sm.flags);
    if (rc) return rc;
  }
  return SAMPLER_OK;
}

int sampler_get_history(sampler* h, int32_t slot, int32_t* n_prompt, int32_t* n_output, int32_t* prompt_out,
                        int32_t* output_out, int32_t* n_unique, int32_t* uniq_ids, int32_t* uniq_counts,
                        int32_t* uniq_in_prompt) {
  if (!h) return SAMPLER_EINVAL;
  if (slot < 0 || slot >= h->cfg.max_batch) return fail(h, SAMPLER_ERANGE, "slot out of range");
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaDeviceSynchronize());
  SlotMeta sm;
  std::vector<int32_t> toks;
  std::vector<UniqEntry> u;
  int rc = read_slot(h, slot, &sm, &toks, &u);
  if (rc) return rc;
  if (n_prompt) *n_prompt = sm.n_prompt;
  if (n_output) *n_output = sm.n_out;
  if (prompt_out) std::copy(toks.begin(), toks.begin() + sm.n_prompt, prompt_out);
  if (output_out) std::copy(toks.begin() + sm.n_prompt, toks.end(), output_out);
  if (n_unique) *n_unique = sm.n_uniq;
  for (size_t i = 0; i < u.size(); ++i) {
    if (uniq_ids) uniq_ids[i] = u[i].id;
    if (uniq_counts) uniq_counts[i] = (int32_t)(u[i].meta >> 1);
    if (uniq_in_prompt) uniq_in_prompt[i] = (int32_t)(u[i].meta & 1u);
  }
  return SAMPLER_OK;
}

int sampler_get_slot_flags(sampler* h, int32_t slot, int32_t* flags) {
  if (!h || !flags) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (slot < 0 || slot >= h->cfg.max_batch) return fail(h, SAMPLER_ERANGE, "slot out of range");
  CK(h, cudaSetDevice(h->cfg.device));
  CK(h, cudaDeviceSynchronize());
  SlotMeta sm;
  CK(h, cudaMemcpy(&sm, h->d_meta + slot, sizeof(sm), cudaMemcpyDeviceToHost));
  *flags = sm.flags;
  return SAMPLER_OK;
}

// ---- launches -----------------------------------------------------------------------
static int check_logits(sampler* h, const void* logits, int64_t ld, int32_t B) {
  if (!logits) return fail(h, SAMPLER_EINVAL, "logits is NULL");
  if (B < 1 || B > h->cfg.max_batch) return fail(h, SAMPLER_EINVAL, "B=%d out of [1, max_batch=%d]", B, h->cfg.max_batch);
  const int esz = (h->cfg.logits_dtype == SAMPLER_BF16) ? 2 : 4;
  if (((uintptr_t)logits) % 16) return fail(h, SAMPLER_EINVAL, "logits must be 16-byte aligned");
  if (ld < h->cfg.vocab_local || (ld * esz) % 16) return fail(h, SAMPLER_EINVAL, "ld must be >= vocab_local and ld*elem %% 16 == 0");
  return SAMPLER_OK;
}

struct LaunchPlan {
  int spr;         // steps (2 KB of one row) per row
  int span;        // steps per CTA
  int rpr;         // CTA record blocks per row
  int64_t nsteps;  // B * spr
  int grid;
};

// Phase A geometry (stream.cuh): equal contiguous spans of the padded step space, one persistent
// CTA per SM; a span is >= one tile (16 steps) and covers at most kMaxSeg - 2 whole rows.
#ifndef SMP_PEN_IN_B_MAXB
#define SMP_PEN_IN_B_MAXB 32
#endif
#ifndef SMP_PEN_IN_B_RESERVE
#define SMP_PEN_IN_B_RESERVE 1
#endif
#ifndef SMP_EXG_MIN
#define SMP_EXG_MIN 1  // smallest cluster size of the exact kernel
#endif
#ifndef SMP_MINSPAN
#define SMP_MINSPAN kTileSteps
#endif
static LaunchPlan plan(const sampler* h, int32_t B) {
  LaunchPlan p;
  p.spr = (int)(h->Vq / kStepVec);
  p.nsteps = (int64_t)B * p.spr;
  int64_t nctas = (int64_t)h->sm_count * kStreamCtasPerSm;
#if SMP_PEN_IN_B_RESERVE
  // small batches: leave B SMs to phase B (its prologue then overlaps this pass; see pen_in_b)
  if (B <= SMP_PEN_IN_B_MAXB && (int64_t)B * 4 <= nctas) nctas -= B;
#endif
  int64_t span = (p.nsteps + nctas - 1) / nctas;
  span = std::max<int64_t>(span, SMP_MINSPAN);
  // phase B merges at most kBT partial records per row (kCW per CTA touching the row): <= 9 CTAs
  span = std::max<int64_t>(span, (p.spr + kBT / kCW - 2) / (kBT / kCW - 1));
  span = std::min<int64_t>(span, (int64_t)(kMaxSeg - 2) * p.spr);
  p.span = (int)span;
  p.grid = (int)((p.nsteps + span - 1) / span);
  p.rpr = (p.spr + p.span - 1) / p.span + 1;
  return p;
}

// small batches: phase A's grid leaves at least B SMs free, so phase B's CTAs are resident while it
// streams and build the penalty hand-off in their prologue (off phase A's critical path)

static int pen_in_b(const sampler* h, int32_t B, const LaunchPlan& lp) {
  return (B <= SMP_PEN_IN_B_MAXB && lp.grid + B <= h->sm_count) ? 1 : 0;
}

static StreamArgs stream_args(sampler* h, const void* logits, int64_t ld, int32_t B, const int32_t* slots,
                              const sampling_params* params_dev, const LaunchPlan& lp) {
  StreamArgs a{};
  a.logits = logits;
  a.ld = ld;
  a.B = B;
  a.V = h->cfg.vocab_size;
  a.voff = h->cfg.vocab_offset;
  a.vloc = h->cfg.vocab_local;
  a.Vq = h->Vq;
  a.spr = lp.spr;
  a.span = lp.span;
  a.rpr = lp.rpr;
  a.nsteps = lp.nsteps;
  a.slots = slots;
  a.params_dev = params_dev;
  a.params_tab = h->d_params;
  a.pen_mode = h->cfg.penalty_mode;
  a.hs = hist_state(h);
  a.parts = h->d_parts;
  a.hand = h->d_hand;
  a.pent = h->d_pent;
  a.gkeys = h->d_gkeys;
  a.trace = h->d_trace;
  a.pen_in_b = pen_in_b(h, B, lp);
  a.early_tiles = a.pen_in_b;
  return a;
}

static int launch_stream(sampler* h, const StreamArgs& a, int grid, cudaStream_t st) {
  if (h->d_trace)
    CK(h, cudaMemsetAsync(h->d_trace, 0, sizeof(uint64_t) * (trace_a_len(h) + 32 * (int64_t)h->cfg.max_batch), st));
  // programmatic dependent launch: the grid may be scheduled while the previous kernel of the
  // stream finishes (the kernel waits for it before touching memory, stream.cuh)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kStreamThreads);
  cfg.dynamicSmemBytes = kStreamSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (h->cfg.logits_dtype == SAMPLER_BF16)
    CK(h, cudaLaunchKernelEx(&cfg, stream_kernel<__nv_bfloat16>, a));
  else
    CK(h, cudaLaunchKernelEx(&cfg, stream_kernel<float>, a));
  return SAMPLER_OK;
}

static SelectArgs select_args(sampler* h, const void* logits, int64_t ld, int32_t B, const int32_t* slots,
                              const sampling_params* params_dev, const uint64_t* seeds, uint64_t step, int append,
                              const RowOut& ro, const LaunchPlan& lp) {
  SelectArgs s{};
  s.logits = logits;
  s.ld = ld;
  s.B = B;
  s.V = h->cfg.vocab_size;
  s.voff = h->cfg.vocab_offset;
  s.vloc = h->cfg.vocab_local;
  s.Vq = h->Vq;
  s.spr = lp.spr;
  s.span = lp.span;
  s.rpr = lp.rpr;
  s.slots = slots;
  s.params_dev = params_dev;
  s.params_tab = h->d_params;
  s.seeds = seeds;
  s.step = step;
  s.step_dev = h->d_step_src;
  s.kcand = h->cfg.max_top_k;
  s.pen_mode = h->cfg.penalty_mode;
  s.mode = 0;
  s.append = append;
  s.pending_ok = 1;
  s.pen_in_b = pen_in_b(h, B, lp);
  s.hs = hist_state(h);
  s.parts = h->d_parts;
  s.hand = h->d_hand;
  s.pent = h->d_pent;
  s.gkeys = h->d_gkeys;
  s.ro = ro;
  s.out_records = nullptr;
  s.out_stride = h->rec_stride;
  s.trace = h->d_trace ? h->d_trace + trace_a_len(h) : nullptr;
  return s;
}

// phase B with programmatic dependent launch: its CTAs may start (prologue) while phase A's last
// CTAs run; griddepcontrol.wait in the kernel orders every read of phase A's outputs
static int launch_select(sampler* h, const SelectArgs& s, int B, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)B);
  cfg.blockDim = dim3(kBT);
  cfg.dynamicSmemBytes = kSelectSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (h->cfg.logits_dtype == SAMPLER_BF16)
    CK(h, cudaLaunchKernelEx(&cfg, select_rows_kernel<__nv_bfloat16>, s));
  else
    CK(h, cudaLaunchKernelEx(&cfg, select_rows_kernel<float>, s));
  return SAMPLER_OK;
}

static MergeArgs merge_args(sampler* h, const int32_t* slots, const sampling_params* params_dev,
                            const uint64_t* seeds, uint64_t step, int append, const RowOut& ro) {
  MergeArgs m{};
  m.records = nullptr;
  m.rec_stride = h->rec_stride;
  m.rank_pitch = 0;
  m.world = 0;
  m.V = h->cfg.vocab_size;
  m.kcand = h->cfg.max_top_k;
  m.slots = slots;
  m.params_dev = params_dev;
  m.params_tab = h->d_params;
  m.seeds = seeds;
  m.step = step;
  m.step_dev = h->d_step_src;
  m.append = append;
  m.hs = hist_state(h);
  m.ro = ro;
  m.trace = h->d_trace ? h->d_trace + trace_a_len(h) : nullptr;
  m.pen_mode = h->cfg.penalty_mode;
  return m;
}

static int launch_merge(sampler* h, const MergeArgs& m, int B, cudaStream_t st) {
  if (m.xp.world == 0) {
    merge_rows_kernel<<<B, kBT, kMergeKernelSmem, st>>>(m);
    CK(h, cudaGetLastError());
    return SAMPLER_OK;
  }
  // peer exchange: programmatic dependent launch after phase 1 (its CTAs trigger at their start, so
  // every phase-1 CTA is resident before a merge CTA spins on a flag)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(kBT);
  cfg.dynamicSmemBytes = kMergeKernelSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(h, cudaLaunchKernelEx(&cfg, merge_rows_kernel, m));
  return SAMPLER_OK;
}

static int do_sample(sampler* h, const void* logits, int64_t ld, int32_t B, const int32_t* slots_dev,
                     const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step, int32_t append,
                     int32_t* tokens, float* logprobs, float* flogprobs, int32_t* status, cudaStream_t st) {
  const LaunchPlan lp = plan(h, B);
  const StreamArgs a = stream_args(h, logits, ld, B, slots_dev, params_dev, lp);
  RowOut ro{tokens, logprobs, flogprobs, status, h->d_info};
  tmark(h, 0, st);
  int rc = launch_stream(h, a, lp.grid, st);
  if (rc) return rc;
  tmark(h, 1, st);
  rc = launch_select(h, select_args(h, logits, ld, B, slots_dev, params_dev, seeds_dev, step, append, ro, lp), B, st);
  if (rc) return rc;
  tmark(h, 2, st);
  h->last_launches = 2;
  // exact multi-pass kernel only if some row can be unresolved by the one-pass candidates
  bool need = params_dev != nullptr;
  if (!need) {
    const int n = slots_dev ? h->cfg.max_batch : B;
    for (int i = 0; i < n && !need; ++i) need = row_may_pend(h->h_params[i], h->cfg.vocab_size, h->cfg.max_top_k);
  }
  if (need) {
    // one cluster of G CTAs per row (every row launched; rows that are not pending exit at once):
    // G = the largest power of two <= 8 with B * G <= 2 resident CTAs per SM (c2: G = 4)
    // bf16: one CTA per SM (the value-key histogram), chunks of <= 65535 elements
    const bool bf = h->cfg.logits_dtype == SAMPLER_BF16;
    const int per_sm = bf ? 1 : 2;
    int G = SMP_EXG_MIN;
    while (G < 8 && (int64_t)B * G * 2 <= (int64_t)per_sm * h->sm_count) G *= 2;
    while (bf && G < 8 && ((int64_t)h->cfg.vocab_local + G - 1) / G > kKhMaxChunk - 127) G *= 2;
    ExactArgs e{};
    e.logits = logits;
    e.ld = ld;
    e.B = B;
    e.V = h->cfg.vocab_size;
    e.voff = h->cfg.vocab_offset;
    e.vloc = h->cfg.vocab_local;
    e.G = G;
    e.Lc = (int)((((int64_t)h->cfg.vocab_local + G - 1) / G + 127) / 128 * 128);
    e.slots = slots_dev;
    e.params_dev = params_dev;
    e.params_tab = h->d_params;
    e.seeds = seeds_dev;
    e.step = step;
    e.step_dev = h->d_step_src;
    e.append = append;
    e.pen_mode = h->cfg.penalty_mode;
    e.hs = a.hs;
    e.ro = ro;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * G));
    cfg.blockDim = dim3(kExThreads);
    cfg.dynamicSmemBytes = bf ? kExactSmemBf16 : kExactSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (h->cfg.logits_dtype == SAMPLER_BF16)
      CK(h, cudaLaunchKernelEx(&cfg, exact_kernel<__nv_bfloat16>, e));
    else
      CK(h, cudaLaunchKernelEx(&cfg, exact_kernel<float>, e));
    tmark(h, 3, st);
    h->last_launches = 3;
  }
  return SAMPLER_OK;
}

int sampler_sample(sampler* h, const void* logits, int64_t ld, int32_t B, const int32_t* slots_dev,
                   const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step,
                   int32_t append_to_history, int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                   int32_t* row_status_dev, void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  int rc = check_logits(h, logits, ld, B);
  if (rc) return rc;
  if (!tokens_dev || !logprobs_dev) return fail(h, SAMPLER_EINVAL, "tokens/logprobs output is NULL");
  if (h->cfg.vocab_local != h->cfg.vocab_size)
    return fail(h, SAMPLER_EINVAL, "sharded handle: use sampler_sample_local + sampler_merge");
  CK(h, cudaSetDevice(h->cfg.device));
  return do_sample(h, logits, ld, B, slots_dev, params_dev, seeds_dev, step, append_to_history, tokens_dev,
                   logprobs_dev, filtered_logprobs_dev, row_status_dev, (cudaStream_t)cuda_stream);
}

int sampler_debug_distribution(sampler* h, const void* logits, int64_t ld, int32_t B, const int32_t* slots_dev,
                               const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step,
                               int32_t* tokens_dev, float* logprobs_dev, float* q_dev, void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  int rc = check_logits(h, logits, ld, B);
  if (rc) return rc;
  if (!tokens_dev || !logprobs_dev || !q_dev) return fail(h, SAMPLER_EINVAL, "output is NULL");
  if (h->cfg.vocab_local != h->cfg.vocab_size) return fail(h, SAMPLER_EINVAL, "sharded handle");
  CK(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  rc = do_sample(h, logits, ld, B, slots_dev, params_dev, seeds_dev, step, 0, tokens_dev, logprobs_dev, nullptr,
                 nullptr, st);
  if (rc) return rc;
  HistState hs = hist_state(h);
  dim3 grid((unsigned)std::min(64, (h->cfg.vocab_local + 255) / 256), (unsigned)B);
  if (h->cfg.logits_dtype == SAMPLER_BF16)
    debug_q_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(logits, ld, h->cfg.vocab_size, h->cfg.vocab_offset,
                                                         h->cfg.vocab_local, slots_dev, params_dev, h->d_params,
                                                         h->cfg.penalty_mode, hs, h->d_info, q_dev);
  else
    debug_q_kernel<float><<<grid, 256, 0, st>>>(logits, ld, h->cfg.vocab_size, h->cfg.vocab_offset,
                                                 h->cfg.vocab_local, slots_dev, params_dev, h->d_params,
                                                 h->cfg.penalty_mode, hs, h->d_info, q_dev);
  CK(h, cudaGetLastError());
  h->last_launches += 1;
  return SAMPLER_OK;
}

int sampler_debug_trace(const sampler* h, uint64_t* host_out, int32_t n) {
  if (!h || !host_out || n < 0) return SAMPLER_EINVAL;
  if (!h->d_trace) return SAMPLER_EUNSUPPORTED;
  const int64_t m = std::min<int64_t>(n, trace_a_len(h) + 32 * (int64_t)h->cfg.max_batch);
  if (cudaMemcpy(host_out, h->d_trace, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost) != cudaSuccess)
    return SAMPLER_ECUDA;
  return SAMPLER_OK;
}

int64_t sampler_record_bytes(const sampler* h, int32_t B) {
  if (!h || B < 0) return -1;
  return h->rec_stride * (int64_t)B;
}

int sampler_sample_local(sampler* h, const void* logits_slice, int64_t ld, int32_t B, const int32_t* slots_dev,
                         const sampling_params* params_dev, void* records_dev, void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  int rc = check_logits(h, logits_slice, ld, B);
  if (rc) return rc;
  if (!records_dev) return fail(h, SAMPLER_EINVAL, "records_dev is NULL");
  if (((uintptr_t)records_dev) % 16) return fail(h, SAMPLER_EINVAL, "records_dev must be 16-byte aligned");
  CK(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const LaunchPlan lp = plan(h, B);
  tmark(h, 0, st);
  rc = launch_stream(h, stream_args(h, logits_slice, ld, B, slots_dev, params_dev, lp), lp.grid, st);
  if (rc) return rc;
  tmark(h, 1, st);
  RowOut ro{nullptr, nullptr, nullptr, nullptr, h->d_info};
  SelectArgs s = select_args(h, logits_slice, ld, B, slots_dev, params_dev, nullptr, 0, 0, ro, lp);
  s.mode = 1;
  s.out_records = (uint8_t*)records_dev;
  rc = launch_select(h, s, B, st);
  if (rc) return rc;
  tmark(h, 2, st);
  h->last_launches = 2;
  return SAMPLER_OK;
}

int sampler_merge(sampler* h, const void* gathered, int32_t world, int32_t B, const int32_t* slots_dev,
                  const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step, int32_t append,
                  int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev, int32_t* row_status_dev,
                  void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  if (!gathered || !tokens_dev || !logprobs_dev) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (world < 1 || world > kMaxRec) return fail(h, SAMPLER_EINVAL, "world must be in [1, %d]", kMaxRec);
  if (B < 1 || B > h->cfg.max_batch) return fail(h, SAMPLER_EINVAL, "B out of range");
  CK(h, cudaSetDevice(h->cfg.device));
  RowOut ro{tokens_dev, logprobs_dev, filtered_logprobs_dev, row_status_dev, h->d_info};
  MergeArgs m = merge_args(h, slots_dev, params_dev, seeds_dev, step, append, ro);
  m.records = (const uint8_t*)gathered;
  m.rank_pitch = h->rec_stride * B;
  m.world = world;
  tmark(h, 0, (cudaStream_t)cuda_stream);
  int rc = launch_merge(h, m, B, (cudaStream_t)cuda_stream);
  if (rc) return rc;
  tmark(h, 1, (cudaStream_t)cuda_stream);
  h->last_launches = 1;
  return SAMPLER_OK;
}

int64_t sampler_resolve_bytes(const sampler* h, int32_t B) {
  if (!h || B < 0) return -1;
  return kResRowBytes * (int64_t)B;
}

int sampler_resolve_round(sampler* h, const void* logits_slice, int64_t ld, int32_t B, const int32_t* slots_dev,
                          const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step, int32_t round,
                          const void* gathered_dev, int32_t world, int32_t rank, void* payload_dev,
                          int32_t append_to_history, int32_t* tokens_dev, float* logprobs_dev,
                          float* filtered_logprobs_dev, int32_t* row_status_dev, int32_t* active_dev,
                          void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  int rc = check_logits(h, logits_slice, ld, B);
  if (rc) return rc;
  if (!payload_dev || !tokens_dev || !logprobs_dev) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (((uintptr_t)payload_dev) % 16 || (gathered_dev && ((uintptr_t)gathered_dev) % 16))
    return fail(h, SAMPLER_EINVAL, "payload / gathered buffers must be 16-byte aligned");
  if (world < 1 || world > kMaxRec) return fail(h, SAMPLER_EINVAL, "world must be in [1, %d]", kMaxRec);
  if (rank < 0 || rank >= world) return fail(h, SAMPLER_EINVAL, "rank out of [0, world)");
  if (round < 0) return fail(h, SAMPLER_EINVAL, "round must be >= 0");
  if (round > 0 && !gathered_dev) return fail(h, SAMPLER_EINVAL, "gathered_dev is NULL for round > 0");
  CK(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  ResolveArgs a{};
  a.logits = (const uint8_t*)logits_slice;
  a.ld = ld;
  a.esize = (h->cfg.logits_dtype == SAMPLER_BF16) ? 2 : 4;
  a.B = B;
  a.V = h->cfg.vocab_size;
  a.kcand = h->cfg.max_top_k;
  a.world = world;
  a.rank = rank;
  a.round = round;
  a.gathered = (const uint8_t*)gathered_dev;
  a.payload = (uint8_t*)payload_dev;
  a.slots = slots_dev;
  a.params_dev = params_dev;
  a.params_tab = h->d_params;
  a.seeds = seeds_dev;
  a.step = step;
  a.step_dev = h->d_step_src;
  a.append = append_to_history;
  a.hs = hist_state(h);
  a.ro = RowOut{tokens_dev, logprobs_dev, filtered_logprobs_dev, row_status_dev, h->d_info};
  a.info = h->d_info;
  a.rs = h->d_rs;
  a.active = active_dev;
  a.pen_mode = h->cfg.penalty_mode;
  if (active_dev) CK(h, cudaMemsetAsync(active_dev, 0, sizeof(int32_t), st));
  tmark(h, 0, st);
  if (h->cfg.logits_dtype == SAMPLER_BF16)
    resolve_kernel<__nv_bfloat16><<<B, kResThreads, 0, st>>>(a);
  else
    resolve_kernel<float><<<B, kResThreads, 0, st>>>(a);
  CK(h, cudaGetLastError());
  tmark(h, 1, st);
  h->last_launches = 1;
  return SAMPLER_OK;
}

int32_t sampler_resolve_max_rounds(void) { return kResMaxRounds; }

// ---- NEXT-2: one-shot peer exchange --------------------------------------------------------
static ExchPeers exch_peers(const sampler* h) {
  ExchPeers x{};
  x.bases = h->d_xbases;
  x.world = h->x_world;
  x.rank = h->x_rank;
  x.row_stride = h->rec_stride;
  x.rank_pitch = h->rec_stride * (int64_t)h->cfg.max_batch;
  x.par_pitch = x.rank_pitch * h->x_world;
  x.flags_off = 2 * x.par_pitch;
  x.nslots = h->cfg.max_batch;
  x.seq = h->d_xseq;
  x.mseq = h->d_xseq + h->cfg.max_batch;
  x.timeout_ns = h->x_timeout_ns;
  return x;
}

int sampler_exchange_init(sampler* h, int32_t world, int32_t rank, uint32_t timeout_ms, void* ipc_handle_out,
                          void** base_out) {
  if (!h) return SAMPLER_EINVAL;
  if (world < 1 || world > kMaxRec) return fail(h, SAMPLER_EINVAL, "world must be in [1, %d]", kMaxRec);
  if (rank < 0 || rank >= world) return fail(h, SAMPLER_EINVAL, "rank out of [0, world)");
  if (h->d_xbuf) return fail(h, SAMPLER_EINVAL, "exchange already initialised on this handle");
  CK(h, cudaSetDevice(h->cfg.device));
  const int64_t Bm = h->cfg.max_batch;
  // [records: 2 parities x world x B_max][flags: world x B_max] then, 256-aligned, the same for the
  // resolve rounds' payloads (NEXT-1 over the peer exchange)
  const int64_t rec_bytes = 2 * (int64_t)world * Bm * h->rec_stride + (int64_t)world * Bm * 4;
  const int64_t res_off = (rec_bytes + 255) / 256 * 256;
  const int64_t bytes = res_off + 2 * (int64_t)world * Bm * kResRowBytes + (int64_t)world * Bm * 4;
  h->x_res_off = res_off;
  if (cudaMalloc((void**)&h->d_xbuf, bytes) != cudaSuccess || cudaMalloc((void**)&h->d_xbases, sizeof(void*) * world) != cudaSuccess ||
      cudaMalloc((void**)&h->d_xseq, 3 * sizeof(uint32_t) * Bm) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, SAMPLER_ENOMEM, "exchange buffer allocation failed");
  }
  CK(h, cudaMemset(h->d_xbuf, 0, bytes));
  CK(h, cudaMemset(h->d_xseq, 0, 3 * sizeof(uint32_t) * Bm));
  h->x_world = world;
  h->x_rank = rank;
  h->x_bytes = bytes;
  h->x_timeout_ns = (uint64_t)(timeout_ms ? timeout_ms : 10000) * 1000000ull;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t ih;
    CK(h, cudaIpcGetMemHandle(&ih, h->d_xbuf));
    memcpy(ipc_handle_out, &ih, sizeof(ih));
  }
  if (base_out) *base_out = h->d_xbuf;
  return SAMPLER_OK;
}

static int exch_upload(sampler* h, const std::vector<uint8_t*>& b) {
  CK(h, cudaMemcpy(h->d_xbases, b.data(), sizeof(void*) * b.size(), cudaMemcpyHostToDevice));
  return SAMPLER_OK;
}

int sampler_exchange_open(sampler* h, const void* ipc_handles) {
  if (!h || !ipc_handles) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (!h->d_xbuf) return fail(h, SAMPLER_EINVAL, "sampler_exchange_init first");
  CK(h, cudaSetDevice(h->cfg.device));
  std::vector<uint8_t*> b(h->x_world);
  for (int q = 0; q < h->x_world; ++q) {
    if (q == h->x_rank) {
      b[q] = h->d_xbuf;
      continue;
    }
    cudaIpcMemHandle_t ih;
    memcpy(&ih, (const uint8_t*)ipc_handles + (size_t)q * sizeof(ih), sizeof(ih));
    void* p = nullptr;
    CK(h, cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
    h->x_opened.push_back(p);
    b[q] = (uint8_t*)p;
  }
  return exch_upload(h, b);
}

int sampler_exchange_set_peers(sampler* h, void* const* bases_host) {
  if (!h || !bases_host) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (!h->d_xbuf) return fail(h, SAMPLER_EINVAL, "sampler_exchange_init first");
  CK(h, cudaSetDevice(h->cfg.device));
  std::vector<uint8_t*> b(h->x_world);
  for (int q = 0; q < h->x_world; ++q) {
    if (!bases_host[q]) return fail(h, SAMPLER_EINVAL, "NULL peer base");
    b[q] = (uint8_t*)bases_host[q];
  }
  if (b[h->x_rank] != h->d_xbuf) return fail(h, SAMPLER_EINVAL, "bases[rank] must be this handle's own buffer");
  return exch_upload(h, b);
}

int sampler_sample_exchange(sampler* h, const void* logits_slice, int64_t ld, int32_t B, const int32_t* slots_dev,
                            const sampling_params* params_dev, const uint64_t* seeds_dev, uint64_t step,
                            int32_t append, int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                            int32_t* row_status_dev, int32_t phases, void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  if (!h->d_xbuf) return fail(h, SAMPLER_EINVAL, "sampler_exchange_init / open first");
  if (phases < 1 || phases > 3) return fail(h, SAMPLER_EINVAL, "phases must be 1, 2 or 3");
  int rc = check_logits(h, logits_slice, ld, B);
  if (rc) return rc;
  if ((phases & 2) && (!tokens_dev || !logprobs_dev)) return fail(h, SAMPLER_EINVAL, "NULL argument");
  CK(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int nk = 0;
  tmark(h, 0, st);
  if (phases & 1) {
    const LaunchPlan lp = plan(h, B);
    rc = launch_stream(h, stream_args(h, logits_slice, ld, B, slots_dev, params_dev, lp), lp.grid, st);
    if (rc) return rc;
    tmark(h, ++nk, st);
    // phases == 3: the merge is fused into the selection kernel (each CTA publishes its row's record,
    // waits for the peers' records of that row and merges them); phases 1 / 2 split it in two launches
    // (fused only when every row's CTA is resident at once — 2 per SM — so no CTA waits for a peer
    // row that its own GPU has not scheduled yet)
    const bool fused = phases == 3 && B <= 2 * h->sm_count;
    RowOut ro{fused ? tokens_dev : nullptr, fused ? logprobs_dev : nullptr, fused ? filtered_logprobs_dev : nullptr,
              fused ? row_status_dev : nullptr, h->d_info};
    SelectArgs s = select_args(h, logits_slice, ld, B, slots_dev, params_dev, seeds_dev, step, fused ? append : 0, ro,
                               lp);
    s.mode = 1;
    s.xp = exch_peers(h);
    s.fuse_merge = fused ? 1 : 0;
    rc = launch_select(h, s, B, st);
    if (rc) return rc;
    tmark(h, ++nk, st);
  }
  if (phases == 2 || (phases == 3 && B > 2 * h->sm_count)) {
    RowOut ro{tokens_dev, logprobs_dev, filtered_logprobs_dev, row_status_dev, h->d_info};
    MergeArgs m = merge_args(h, slots_dev, params_dev, seeds_dev, step, append, ro);
    m.xp = exch_peers(h);
    m.records = h->d_xbuf;
    m.rank_pitch = m.xp.rank_pitch;
    m.world = h->x_world;
    rc = launch_merge(h, m, B, st);
    if (rc) return rc;
    tmark(h, ++nk, st);
  }
  h->last_launches = nk;
  return SAMPLER_OK;
}

int sampler_set_step_source(sampler* h, const uint64_t* step_dev) {
  if (!h) return SAMPLER_EINVAL;
  if (step_dev && ((uintptr_t)step_dev) % 8) return fail(h, SAMPLER_EINVAL, "step_dev must be 8-byte aligned");
  h->d_step_src = step_dev;
  return SAMPLER_OK;
}

static ExchPeers exch_peers_resolve(const sampler* h) {
  ExchPeers x = exch_peers(h);
  x.row_stride = kResRowBytes;
  x.rank_pitch = kResRowBytes * (int64_t)h->cfg.max_batch;
  x.par_pitch = x.rank_pitch * h->x_world;
  x.flags_off = 2 * x.par_pitch;
  x.region_off = h->x_res_off;
  x.seq = h->d_xseq + 2 * h->cfg.max_batch;
  x.mseq = nullptr;
  return x;
}

int sampler_resolve_round_exchange(sampler* h, const void* logits_slice, int64_t ld, int32_t B,
                                   const int32_t* slots_dev, const sampling_params* params_dev,
                                   const uint64_t* seeds_dev, uint64_t step, int32_t round, int32_t append_to_history,
                                   int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                                   int32_t* row_status_dev, int32_t* active_dev, void* cuda_stream) {
  if (!h) return SAMPLER_EINVAL;
  if (!h->d_xbuf) return fail(h, SAMPLER_EINVAL, "sampler_exchange_init / open first");
  int rc = check_logits(h, logits_slice, ld, B);
  if (rc) return rc;
  if (!tokens_dev || !logprobs_dev) return fail(h, SAMPLER_EINVAL, "NULL argument");
  if (round < 0) return fail(h, SAMPLER_EINVAL, "round must be >= 0");
  CK(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  ResolveArgs a{};
  a.logits = (const uint8_t*)logits_slice;
  a.ld = ld;
  a.esize = (h->cfg.logits_dtype == SAMPLER_BF16) ? 2 : 4;
  a.B = B;
  a.V = h->cfg.vocab_size;
  a.kcand = h->cfg.max_top_k;
  a.world = h->x_world;
  a.rank = h->x_rank;
  a.round = round;
  a.slots = slots_dev;
  a.params_dev = params_dev;
  a.params_tab = h->d_params;
  a.seeds = seeds_dev;
  a.step = step;
  a.step_dev = h->d_step_src;
  a.append = append_to_history;
  a.hs = hist_state(h);
  a.ro = RowOut{tokens_dev, logprobs_dev, filtered_logprobs_dev, row_status_dev, h->d_info};
  a.info = h->d_info;
  a.rs = h->d_rs;
  a.active = active_dev;
  a.pen_mode = h->cfg.penalty_mode;
  a.rx = exch_peers_resolve(h);
  if (active_dev) CK(h, cudaMemsetAsync(active_dev, 0, sizeof(int32_t), st));
  tmark(h, 0, st);
  if (h->cfg.logits_dtype == SAMPLER_BF16)
    resolve_kernel<__nv_bfloat16><<<B, kResThreads, 0, st>>>(a);
  else
    resolve_kernel<float><<<B, kResThreads, 0, st>>>(a);
  CK(h, cudaGetLastError());
  tmark(h, 1, st);
  h->last_launches = 1;
  return SAMPLER_OK;
}

}  // extern "C"

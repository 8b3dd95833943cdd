/*
 * sampler.h — C ABI of the B200-native last-stage sampler (arXiv 2506.22033, "SiPipe").
 *
 * The operation: turn a batch of decode logits Z[B x V] into next tokens, per row b:
 *
 *   p_b = Filter( softmax( ApplyPenalty(z_b, y_<s) / tau ) ; k, p )      PAPER.md P:150-158 (§2.1, eq.)
 *   y_b ~ Categorical(p_b)                                               PAPER.md P:161 (§2.1 step 3)
 *   Z' = Z - alpha*f, f = CalcPenalty(Y) (frequency / presence / repetition)  P:354 (§5.1)
 *   Z'' = Z'/tau,  P_ij = exp(Z''_ij) / sum_v exp(Z''_iv)                P:354 (§5.1)
 *   top-k / top-p restrict candidates; min-p is listed at P:529 (§7.1)
 *   incremental per-request history, "only the B elements ... updated"  P:368-371 (§5.1 (1),(2))
 *   TP logits shards B x V/t combined without an all-gather of logits   P:375 (§5.1 (3))
 *
 * Exact semantics (tie-breaks, filter order, RNG, penalty rounding, greedy epsilon) are the
 * readings R1..R15 of DESIGN.md §3 (= SURVEY.md §8(c)); the float64 oracle in oracle/ is the
 * executable statement of them.  The interface follows SPEC.md's sampler module
 * (SamplingParams S:146-149, SamplingOutput S:151-154, new_replica/append/evict_and_admit
 * S:157-195, sample S:227-235, errors S:161/S:181/S:209, ownership S:264).
 *
 * Conventions
 *  - Every function returns int32 status: SAMPLER_OK (0) or a negative SAMPLER_E* code.
 *    On error, sampler_last_error(h) holds a one-line message.  Argument / range errors
 *    are detected on the host BEFORE any launch and have no side effects.
 *  - "dev" pointers are CUDA device pointers of the handle's device; "host" pointers are
 *    ordinary host memory.  Nothing is retained after a call returns except by the handle.
 *  - Calls marked ASYNC are stream-ordered on `cuda_stream` (a cudaStream_t; NULL = legacy
 *    default stream): they only enqueue kernels, and every borrowed buffer must stay alive
 *    and unmodified until the stream has passed the call.  Calls marked SYNC return after the
 *    device work they issue has completed.
 *  - A handle has ONE owner thread at a time.  Handles are independent.
 *  - Logits are row-major [B x ld] (bf16 or fp32), row b at logits + b*ld elements.  Required:
 *    logits 16-byte aligned, ld*sizeof(elem) % 16 == 0, ld >= vocab_local, and the buffer
 *    readable for B*ld elements (rows are streamed with 16-byte bulk copies).  Logits are
 *    borrowed read-only: the library never writes them (unlike the paper's in-place CPU
 *    layout).
 *  - Data-dependent row faults (a NaN or +inf logit; a row whose every logit is -inf) never
 *    fail the call: that row gets token -1, logprob NaN and a non-zero row_status.
 *    -inf logits are legal and mean probability 0.
 */
#ifndef PAPER_2506_22033_B200_SAMPLER_H
#define PAPER_2506_22033_B200_SAMPLER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------- */
enum {
  SAMPLER_OK = 0,
  SAMPLER_EINVAL = -1,       /* bad argument (NULL handle/pointer, bad size/alignment, bad param) */
  SAMPLER_ENOMEM = -2,       /* device allocation failed */
  SAMPLER_ECUDA = -3,        /* a CUDA runtime call or launch failed (message has the CUDA error) */
  SAMPLER_ERANGE = -4,       /* token id outside [0,V), slot outside [0,B_max), history > L_max */
  SAMPLER_EUNSUPPORTED = -5  /* valid but unsupported request (e.g. dtype, vocab > 2^31-2^20) */
};

/* logits dtype codes */
enum { SAMPLER_F32 = 0, SAMPLER_BF16 = 2 };

/* penalty semantics (R1):
 *  OPENAI_CTRL: for ids with cnt>0 or in-prompt: y=x; if r!=1: y = y>0 ? y/r : y*r;
 *               if cnt>0: y = y - freq*cnt; y = y - pres     (each op rounded to binary32)
 *  LINEAR     : paper-literal Z' = Z - alpha*f:
 *               y = ((x - freq*cnt) - pres*[cnt>0]) - rep*[cnt>0 or in-prompt]
 *               where `repetition_penalty` is used as the subtractive coefficient alpha_rep. */
enum { SAMPLER_PEN_OPENAI_CTRL = 0, SAMPLER_PEN_LINEAR = 1 };

/* per-row status written to row_status_dev */
enum {
  SAMPLER_ROW_OK = 0,
  SAMPLER_ROW_NONFINITE = 1,   /* a NaN or +inf logit in the row ("finite entries") */
  SAMPLER_ROW_ALL_NEG_INF = 2, /* no token has positive probability */
  SAMPLER_ROW_UNRESOLVED = 3,  /* vocab-sharded merge: the row's kept set is not bounded by the
                                  exchanged candidates (top-p/min-p-only rows, or top_k >
                                  max_top_k); the sampler_resolve_round rounds below finish it
                                  (DESIGN.md §8 NEXT-1).  Never produced by sampler_sample on an
                                  unsharded handle. */
  SAMPLER_ROW_INVALID = 4,     /* slots_dev[b] outside [0, B_max), or params_dev[b] a parameter set
                                  that sampler_set_params would reject: checked on the device, the
                                  row gets token -1 and logprob NaN, its slot is not touched */
  SAMPLER_ROW_EXCHANGE_TIMEOUT = 5 /* sampler_sample_exchange: a peer's record for this row did not
                                  arrive within the handle's timeout (a rank stopped calling);
                                  token -1, logprob NaN, no append — the GPU is never hung */
};

typedef struct {
  int32_t vocab_size;     /* V: global vocabulary size, 1 <= V <= 2^31 - 2^20 */
  int32_t vocab_offset;   /* first global id of this rank's slice (0 when unsharded) */
  int32_t vocab_local;    /* slice length (== vocab_size when unsharded); ids
                             [vocab_offset, vocab_offset+vocab_local) are local */
  int32_t max_batch;      /* B_max: number of request slots (rows per call <= B_max) */
  int32_t max_history;    /* L_max: prompt + output tokens per slot */
  int32_t max_top_k;      /* K_cand in [1, 128]: candidates kept per partial reduction.  Rows
                             with 1 <= top_k <= K_cand (and greedy rows) are always exact in one
                             streaming pass; other rows take the exact multi-pass path. */
  int32_t logits_dtype;   /* SAMPLER_F32 | SAMPLER_BF16 */
  int32_t penalty_mode;   /* SAMPLER_PEN_* */
  int32_t device;         /* CUDA device ordinal; the handle's memory lives there */
} sampler_config;

/* Per-row sampling parameters.  48 bytes, 8-byte aligned; the same layout
 * is used for host arrays (set_params) and device arrays (params_dev). */
typedef struct {
  float temperature;        /* >= 0; < 1e-5 (incl. 0) => greedy (R5); < 0 => EINVAL */
  int32_t top_k;            /* <= 0 or >= V => off; k => keep the k best (z' desc, id asc) */
  float top_p;              /* in (0, 1]; 1 => off */
  float min_p;              /* in [0, 1]; 0 => off; keep p >= min_p * p_max */
  float repetition_penalty; /* OPENAI_CTRL: > 0, 1 => off.  LINEAR: alpha_rep, 0 => off */
  float presence_penalty;   /* 0 => off (any finite value) */
  float frequency_penalty;  /* 0 => off (any finite value) */
  int32_t reserved;         /* must be 0 */
  uint64_t seed;            /* Philox key (R11) */
  uint64_t request_id;      /* Philox counter words 2-3: keys the draw by request, not row */
} sampling_params;

typedef struct sampler sampler; /* opaque handle */

/* ---- lifecycle ---------------------------------------------------------------------- */

/* SYNC.  Validate cfg, allocate all device state on cfg->device (params table, per-slot
 * history store and unique-token penalty table [B_max x L_max], workspace) and return the
 * handle in *out.  All slots start with empty history and default params (greedy off,
 * temperature 1, no filters, no penalties, seed 0, request_id = slot).
 * Errors: EINVAL (NULL args, sizes out of range), ENOMEM, ECUDA.  On error *out = NULL. */
int sampler_create(const sampler_config* cfg, sampler** out);

/* SYNC.  Free everything the handle owns.  NULL is a no-op returning OK. */
int sampler_destroy(sampler* h);

/* Message describing the last failing call on h ("" if none).  Valid until the next call on
 * h.  With h == NULL: the message of the last failing sampler_create on this thread. */
const char* sampler_last_error(const sampler* h);

/* ---- per-slot state ----------------------------------------------------------------- */

/* SYNC.  Waits for all work on the handle's device (an in-flight sample may still read the table),
 * then copies n host params into the handle's table at host slot indices slots[0..n).
 * Every entry is validated first (EINVAL: temperature < 0 or non-finite, top_p not in
 * (0,1], min_p not in [0,1], repetition_penalty <= 0 in OPENAI_CTRL mode, non-finite
 * penalties, reserved != 0; ERANGE: slot outside [0, B_max)); nothing is written on error. */
int sampler_set_params(sampler* h, int32_t n, const int32_t* slots_host,
                       const sampling_params* params_host);

/* SYNC.  Waits for all work on the handle's device (an in-flight sample with append may still write
 * the slot), then admits / evicts (SPEC S:187 evict_and_admit): replaces slot's history with the given
 * host token lists and rebuild its unique-token penalty table from scratch.
 * prompt/output may be NULL when their count is 0.
 * Errors: ERANGE (slot out of range, n_prompt + n_output > L_max, any id outside [0, V)). */
int sampler_set_history(sampler* h, int32_t slot, const int32_t* prompt_host, int32_t n_prompt,
                        const int32_t* output_host, int32_t n_output);

/* SYNC.  Append one output token to each of n slots (SPEC S:177 append_tokens): the slot's
 * output list grows by one and its penalty entry is updated incrementally.
 * Errors: ERANGE (slot, token or L_max overflow) — checked for all n before any change. */
int sampler_append_tokens(sampler* h, int32_t n, const int32_t* slots_host,
                          const int32_t* tokens_host);

/* SYNC.  Export a slot's state for inspection / checkpoint.  Any output pointer may be NULL.
 *  n_prompt, n_output: history lengths; prompt_out/output_out: capacity >= L_max tokens;
 *  n_unique + uniq_ids/uniq_counts/uniq_in_prompt (capacity >= L_max): the incremental
 *  penalty table (ids ascending; counts = occurrences in the output; in_prompt 0/1). */
int sampler_get_history(sampler* h, int32_t slot, int32_t* n_prompt, int32_t* n_output,
                        int32_t* prompt_out, int32_t* output_out, int32_t* n_unique,
                        int32_t* uniq_ids, int32_t* uniq_counts, int32_t* uniq_in_prompt);

/* SYNC.  The slot's status bits in *flags: SAMPLER_SLOT_OVERFLOW (bit 0) = an in-kernel append
 * found the history at L_max and dropped the token (sticky until sampler_set_history).
 * Errors: EINVAL (NULL), ERANGE (slot out of range). */
enum { SAMPLER_SLOT_OVERFLOW = 1 };
int sampler_get_slot_flags(sampler* h, int32_t slot, int32_t* flags);

/* ---- sampling ----------------------------------------------------------------------- */

/* ASYNC.  Sample one token for each of B rows of logits (unsharded handle:
 * vocab_local == vocab_size).
 *  logits      dev [B x ld] of cfg->logits_dtype (see alignment rules above)
 *  slots_dev   dev int32[B]: row b uses request slot slots_dev[b] (distinct); NULL => b
 *  params_dev  dev sampling_params[B] for row b; NULL => the slot's table entry (set_params)
 *  seeds_dev   dev uint64[B]: overrides params.seed for row b; NULL => params.seed
 *  step        Philox counter words 0-1 (decode step)
 *  append_to_history  nonzero => append each sampled token to its slot; rows
 *              with a non-OK status append nothing.  Overflowing L_max sets the slot's
 *              overflow bit (SAMPLER_SLOT_OVERFLOW, read with sampler_get_slot_flags) and appends nothing.
 *  tokens_dev  dev int32[B] out; logprobs_dev dev float[B] out = log softmax(z'/tau_eff)[tok]
 *              (full vocabulary, before filtering; R12)
 *  filtered_logprobs_dev  dev float[B] out, nullable: log of the token's probability in the
 *              final filtered, renormalised distribution (0 for greedy rows)
 *  row_status_dev  dev int32[B] out, nullable: SAMPLER_ROW_*
 * Errors: EINVAL (NULL handle/logits/tokens/logprobs, B < 1 or > B_max, bad alignment, sharded
 * handle), ECUDA. */
int sampler_sample(sampler* h, const void* logits, int64_t ld, int32_t B,
                   const int32_t* slots_dev, const sampling_params* params_dev,
                   const uint64_t* seeds_dev, uint64_t step, int32_t append_to_history,
                   int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                   int32_t* row_status_dev, void* cuda_stream);

/* ASYNC, test/debug only.  Same inputs as sampler_sample (no history append); additionally
 * writes q_dev [B x vocab_size] fp32 = the final filtered distribution (w_v / W for kept ids,
 * 0 elsewhere; one-hot for greedy rows).  For parity tests on small shapes. */
int sampler_debug_distribution(sampler* h, const void* logits, int64_t ld, int32_t B,
                               const int32_t* slots_dev, const sampling_params* params_dev,
                               const uint64_t* seeds_dev, uint64_t step,
                               int32_t* tokens_dev, float* logprobs_dev, float* q_dev,
                               void* cuda_stream);

/* ---- vocab-sharded two-phase sampling (TP-style logits shards) ---------------- */

/* Bytes of one rank's candidate records for B rows (the all-gather payload per rank). */
int64_t sampler_record_bytes(const sampler* h, int32_t B);

/* ASYNC.  Phase 1 on this rank's slice logits_slice [B x ld] (ids vocab_offset + j):
 * penalties for local ids, local max / sum and the local top-K_cand candidates per row, written
 * to records_dev (sampler_record_bytes(h,B) bytes, device).  The caller all-gathers the records
 * of all ranks (rank order) and calls sampler_merge. */
int sampler_sample_local(sampler* h, const void* logits_slice, int64_t ld, int32_t B,
                         const int32_t* slots_dev, const sampling_params* params_dev,
                         void* records_dev, void* cuda_stream);

/* ASYNC.  Phase 2: merge `world` ranks' records (gathered_records_dev = world consecutive
 * blocks of sampler_record_bytes(h,B) bytes, rank order) into the final tokens.  Every rank
 * computes identical outputs (deterministic, rank-ordered reductions).  History append (if
 * requested) is applied on every rank (replicated per-rank tables).  Rows whose kept set is not
 * bounded by the candidates get SAMPLER_ROW_UNRESOLVED (token -1, no append) and are finished by
 * the resolve rounds below. */
int sampler_merge(sampler* h, const void* gathered_records_dev, int32_t world, int32_t B,
                  const int32_t* slots_dev, const sampling_params* params_dev,
                  const uint64_t* seeds_dev, uint64_t step, int32_t append_to_history,
                  int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                  int32_t* row_status_dev, void* cuda_stream);

/* ---- vocab-sharded rows not bounded by the candidates (NEXT-1) ------------------------
 * The filter is over the whole renormalised distribution (§2.1 eq.), so a top-p-only,
 * min-p-only or unfiltered row (or top_k > max_top_k) needs more than the candidate records.  Such
 * a row is finished, without gathering logits (§5.1 (3)), by a distributed mass-weighted
 * radix select over the pi-order keys (z' desc, id asc): per round every rank histograms its slice
 * (256 bins of the next 8 key bits: counts and 128-bit fixed-point masses w*2^80) or, once the
 * target bin holds <= 638 elements, sends those elements; every rank ingests the same gathered
 * bytes with integer arithmetic and narrows the same per-row state (top-k cutoff, then top-p
 * cutoff, then the kept mass per rank, then the owner rank's id-order draw; min-p is an
 * element-wise test).  DESIGN.md §8 (NEXT-1) has the protocol.
 *
 * Usage, after sampler_merge on every rank (same B / slots / params / seeds / step):
 *   round 0: sampler_resolve_round(..., round=0, gathered=NULL, ...) -> payload
 *   round r = 1, 2, ...: all-gather the payloads (rank order, world x sampler_resolve_bytes(h,B)
 *            bytes) and call sampler_resolve_round(..., round=r, gathered, ...) -> next payload;
 *   stop when *active_dev == 0 after a round (or after sampler_resolve_max_rounds() exchanges,
 *   which always suffices: capturable in a CUDA graph with a fixed round count).
 * Resolved rows get their token / logprobs / status SAMPLER_ROW_OK written into the same output
 * arrays as sampler_merge (and the history append, on every rank, when append_to_history); rows
 * the merge already decided are not touched.  Rows still unresolved (too few rounds) keep
 * SAMPLER_ROW_UNRESOLVED.  The handle keeps one state per row between rounds: one resolve sequence
 * per handle at a time, stream-ordered (ASYNC).
 * Errors: EINVAL (NULL / misaligned buffers, world not in [1,16], rank not in [0,world), round < 0,
 * gathered NULL for round > 0), ECUDA. */

/* Bytes of one rank's resolve payload for B rows (16 + 5120 per row). */
int64_t sampler_resolve_bytes(const sampler* h, int32_t B);

/* ASYNC.  One resolve round on this rank (see above).  logits_slice / ld as for
 * sampler_sample_local; gathered_dev: the previous round's all-gathered payloads (dev, world x
 * resolve_bytes, rank order; NULL at round 0); payload_dev (dev, resolve_bytes(h,B), 16-byte
 * aligned): this round's payload; outputs as for sampler_merge; active_dev (dev int32, nullable):
 * set to the number of rows still unresolved after this round. */
int sampler_resolve_round(sampler* h, const void* logits_slice, int64_t ld, int32_t B,
                          const int32_t* slots_dev, const sampling_params* params_dev,
                          const uint64_t* seeds_dev, uint64_t step, int32_t round,
                          const void* gathered_dev, int32_t world, int32_t rank, void* payload_dev,
                          int32_t append_to_history, int32_t* tokens_dev, float* logprobs_dev,
                          float* filtered_logprobs_dev, int32_t* row_status_dev,
                          int32_t* active_dev, void* cuda_stream);

/* Exchanges after which every row is resolved (2 x (8 histogram + 1 gather) + kept mass + draw). */
int32_t sampler_resolve_max_rounds(void);

/* ---- NEXT-2: one-shot peer exchange (NVLink P2P stores + flags, no collective call) ----------
 * The vocab-sharded step of sampler_sample_local -> all-gather -> sampler_merge as ONE call per
 * rank with no NCCL launch: phase 1's epilogue stores each row's candidate record straight into
 * every rank's exchange buffer (P2P stores over NVLink / NVSwitch through IPC-mapped pointers) and
 * raises a per-(rank, row) flag there (system-scope release); the merge kernel waits for every
 * rank's flag of its row (acquire) and merges its local copies.  Records are double-buffered by a
 * per-row sequence number (parity), the TSEM versioned-buffer idea (§5.2): no host
 * synchronisation and no per-step host argument change, so the whole step replays from one CUDA
 * graph.  Every rank must make the same sequence of sampler_sample_exchange calls (same B).
 * Rows the candidates do not bound still get SAMPLER_ROW_UNRESOLVED (finish them with the resolve
 * rounds above). */

/* SYNC.  Allocate this rank's exchange buffer (2 x world x max_batch x record stride bytes of
 * records + world x max_batch u32 flags, zeroed) on the handle's device.  ipc_handle_out (host,
 * nullable, 64 bytes = cudaIpcMemHandle_t) receives the buffer's IPC handle for the peers;
 * base_out (host, nullable) its device address.  timeout_ms: how long a merge waits for a peer
 * before reporting SAMPLER_ROW_EXCHANGE_TIMEOUT (0 => 10000).  Errors: EINVAL (world not in
 * [1,16], rank not in [0,world), already initialised), ENOMEM, ECUDA. */
int sampler_exchange_init(sampler* h, int32_t world, int32_t rank, uint32_t timeout_ms,
                          void* ipc_handle_out, void** base_out);

/* SYNC.  Map every peer's buffer from the world x 64 bytes of IPC handles (host, rank order; this
 * rank's own entry is ignored) with cudaIpcOpenMemHandle (peer access enabled lazily).  The
 * mappings are closed by sampler_destroy.  Errors: EINVAL, ECUDA (a handle could not be opened). */
int sampler_exchange_open(sampler* h, const void* ipc_handles);

/* SYNC.  Alternative to sampler_exchange_open for buffers already addressable in this process (several
 * handles of one process, or mappings the caller made): bases_host[q] = rank q's buffer as returned
 * by its sampler_exchange_init base_out; bases_host[rank] must be this handle's own. */
int sampler_exchange_set_peers(sampler* h, void* const* bases_host);

/* ASYNC.  The vocab-sharded step through the peer exchange.  Arguments as sampler_sample_local +
 * sampler_merge.  phases: 1 = local pass + publish (no outputs), 2 = wait + merge, 3 = both (the
 * normal call; 1 and 2 let several ranks of ONE process and GPU run in lock step without any kernel
 * waiting on a kernel queued behind it).  With phases = 3 and B <= 2 x the SM count the merge is
 * fused into the selection kernel (each CTA publishes its row's record, waits for the peers' records
 * of that row and merges them: two launches per step); larger batches use the separate merge kernel. */
int sampler_sample_exchange(sampler* h, const void* logits_slice, int64_t ld, int32_t B,
                            const int32_t* slots_dev, const sampling_params* params_dev,
                            const uint64_t* seeds_dev, uint64_t step, int32_t append_to_history,
                            int32_t* tokens_dev, float* logprobs_dev, float* filtered_logprobs_dev,
                            int32_t* row_status_dev, int32_t phases, void* cuda_stream);

/* ASYNC.  One resolve round (sampler_resolve_round, NEXT-1) through the peer exchange instead of a
 * caller all-gather: the previous round's payloads are read from this rank's exchange buffer once
 * every rank's flag for the row has arrived (bounded wait: SAMPLER_ROW_EXCHANGE_TIMEOUT), and this
 * round's payload is stored into every rank's buffer with the row's flag raised.  Rounds 0, 1, 2, ...
 * follow sampler_sample_exchange (or sampler_merge) on every rank, exactly as with
 * sampler_resolve_round but with no collective call in between; the round count rule is the same. */
int sampler_resolve_round_exchange(sampler* h, const void* logits_slice, int64_t ld, int32_t B,
                                   const int32_t* slots_dev, const sampling_params* params_dev,
                                   const uint64_t* seeds_dev, uint64_t step, int32_t round,
                                   int32_t append_to_history, int32_t* tokens_dev, float* logprobs_dev,
                                   float* filtered_logprobs_dev, int32_t* row_status_dev,
                                   int32_t* active_dev, void* cuda_stream);

/* ---- per-step parameters on the device (CUDA-graph replays of a decode loop) ----------------
 * The TSEM idea of versioned per-step inputs (§5.2): with step_dev != NULL (device
 * uint64, 8-byte aligned, owned by the caller and alive while calls use it), every later sample /
 * merge / sample_exchange / resolve_round call reads the Philox step (R11) from *step_dev
 * when its kernels run and ignores its host `step` argument.  A decode step captured once in a CUDA
 * graph then samples a new step per replay when the caller advances *step_dev (for instance with an
 * increment captured in the same graph).  NULL restores the host argument.  No synchronisation.
 * Errors: EINVAL (NULL handle, misaligned pointer). */
int sampler_set_step_source(sampler* h, const uint64_t* step_dev);

/* ---- introspection ------------------------------------------------------------------ */

/* Number of kernel launches the last sample / sample_local / merge / debug call enqueued. */
int32_t sampler_last_launch_count(const sampler* h);

/* SYNC, debug only.  With the environment variable SAMPLER_TRACE set at sampler_create, the
 * streaming kernel records per-CTA phase timestamps (globaltimer, ns; 32 slots per CTA) of the
 * last launch; copies min(n, 32 * CTAs) of them to host_out.  EUNSUPPORTED when tracing is off. */
int sampler_debug_trace(const sampler* h, uint64_t* host_out, int32_t n);

/* Per-kernel timing (measurement support).  sampler_set_timing(h, 1) makes every subsequent
 * sample / sample_local / merge call record CUDA events on its stream around each kernel it
 * launches (do not enable while capturing a CUDA graph).  sampler_kernel_times (SYNC: waits for
 * the last call's final event) writes the last call's per-kernel durations in milliseconds, in
 * launch order, to ms_out[0..min(n, count)) and the kernel count to *count.  EINVAL when timing
 * is off or nothing was timed yet. */
int sampler_set_timing(sampler* h, int32_t enable);
int sampler_kernel_times(sampler* h, float* ms_out, int32_t n, int32_t* count);

/* Build identification string (arch, compile flags). */
const char* sampler_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_2506_22033_B200_SAMPLER_H */

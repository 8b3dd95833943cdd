"""Float64 CPU oracle of the last-stage sampling task — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
arm may import, call or execute anything under oracle/.  The product path
(paper_2506_22033_b200/) never imports it, shares no code, header, table or helper
with it, and fails loudly when its CUDA library is missing.

What it computes is the paper's definition of sampling, one row at a time, plainly:

    p = Filter( softmax( ApplyPenalty(z, y_<s) / tau ) ; k, p )        PAPER.md P:150-158 (§2.1 eq.)
    y ~ Categorical(p)                                                   PAPER.md P:161 (§2.1 step 3)
    Z' = Z - alpha * f,  f = CalcPenalty(Y) (frequency/presence/repetition)  P:354 (§5.1)
    softmax P_ij = exp(Z''_ij) / sum_v exp(Z''_iv),  Z'' = Z'/tau        P:354 (§5.1)

Where the paper is silent or ambiguous this file follows the readings listed in
DESIGN.md §3 (R1..R15, = SURVEY.md §8(c)); each step below names its reading.

Every step is float64 except the penalty step, which emulates binary32 with
"one float64 op, then round to float32" (exact emulation since 53 >= 2*24+2),
because the penalised logits z' are the selection keys (R3).

Pinned by tests/test_oracle.py (Philox KATs, SPEC hand values, closed forms,
brute force on tiny vocabularies, chi-squared of draws against the closed-form
softmax, library cross-checks).  No function here is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .philox import uniform as philox_uniform

# penalty modes (R1)
PEN_OPENAI_CTRL = 0
PEN_LINEAR = 1

# row status codes (R15; "all-(-inf) column rejected")
ROW_OK = 0
ROW_NONFINITE = 1   # a NaN or +inf logit in the row
ROW_ALL_NEG_INF = 2  # no token has positive weight

GREEDY_EPS = 1e-5    # DESIGN.md R5: tau < 1e-5 (incl. 0) => greedy
FLAG_EPS = 1e-6      # north star: "within 1e-6 of a CDF or tie boundary" (reported: RowResult.flagged6)
FLAG_EPS_GPU = 1e-10  # DESIGN.md R16: the excuse band actually applied (RowResult.flagged).  Both sides
                      # compute kept-set weights and prefix sums in float64: this oracle's sequential
                      # cumsum is within n * 2^-53 * W (< 2.3e-11 W for n <= 2e5 terms) of the exact sum,
                      # the GPU's bucketed fixed-point masses within 5e-13 W, so a token may differ only
                      # when a boundary lies within ~2.5e-11 W of it; the band is 4x that.  The north
                      # star's 1e-6 is its upper limit, not its value (at 1e-6 a 1e5-token nucleus is
                      # flagged in ~20% of draws, against the < 1e-4 bar; reported as flagged6)


@dataclass
class Params:
    """Per-row sampling parameters (SPEC S:146-149 SamplingParams)."""
    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0
    min_p: float = 0.0
    repetition_penalty: float = 1.0
    presence_penalty: float = 0.0
    frequency_penalty: float = 0.0
    seed: int = 0
    request_id: int = 0


@dataclass
class RowResult:
    token: int
    logprob: float
    filtered_logprob: float
    status: int
    flagged: bool
    greedy: bool
    M: float = float("nan")
    S: float = float("nan")
    u: float = float("nan")
    kept: np.ndarray | None = None        # K3, ascending ids
    q: np.ndarray | None = None           # final filtered distribution over V
    flags: dict = field(default_factory=dict)       # band FLAG_EPS_GPU (the excuse; R16)
    flagged6: bool = False                          # any boundary within FLAG_EPS (north star literal)
    flags6: dict = field(default_factory=dict)


def f32(x):
    """Round a float64 scalar/array to the nearest binary32 (ties-to-even)."""
    return np.float32(x) if np.isscalar(x) else np.asarray(x, dtype=np.float64).astype(np.float32)


# --------------------------------------------------------------------------- decode
def decode_logits(raw, dtype: str) -> np.ndarray:
    """Step 1: logits -> float64 exactly.

    dtype 'f32': raw is float32.  dtype 'bf16': raw is uint16 bit patterns;
    bf16 bits << 16 is the binary32 with the same value (exact)."""
    raw = np.asarray(raw)
    if dtype == "f32":
        return raw.astype(np.float32).astype(np.float64)
    if dtype == "bf16":
        bits = raw.astype(np.uint16).astype(np.uint32) << np.uint32(16)
        return bits.view(np.float32).astype(np.float64)
    raise ValueError(dtype)


# --------------------------------------------------------------------------- penalties
def history_counts(prompt, output, vocab):
    """cnt_v = occurrences of v in the output; inP_v = v in the prompt.

    Frequency/presence use output tokens only, repetition uses prompt ∪ output
    (R2; SPEC S:143 / S:273)."""
    cnt = np.zeros(vocab, dtype=np.int64)
    for t in output:
        cnt[int(t)] += 1
    inp = np.zeros(vocab, dtype=bool)
    for t in prompt:
        inp[int(t)] = True
    return cnt, inp


def apply_penalties(z32: np.ndarray, prompt, output, p: Params, mode: int = PEN_OPENAI_CTRL,
                    vocab_offset: int = 0, vocab: int | None = None) -> np.ndarray:
    """Step 2: Z' = ApplyPenalty(Z, y_<s)  (§2.1(1); §5.1).

    z32: float32 logits of ids [vocab_offset, vocab_offset+len(z32)).
    Every arithmetic op is one float64 op rounded to binary32 (R3).

    OPENAI_CTRL (R1, default): for v with cnt_v>0 or inP_v
        y = x_v
        if r != 1: y = f32(y / r) if y > 0 else f32(y * r)
        if cnt_v > 0: y = f32(y - f32(freq*cnt_v)); y = f32(y - pres)
    LINEAR (paper-literal Z - alpha*f):
        y = f32(f32(f32(x - f32(a_f*cnt)) - a_p*[cnt>0]) - a_r*[cnt>0 or inP])
        with a_r = repetition_penalty used as a subtractive coefficient.
    """
    z = np.array(z32, dtype=np.float32, copy=True)
    n = len(z)
    V = vocab if vocab is not None else vocab_offset + n
    cnt, inp = history_counts(prompt, output, V)
    r = float(np.float32(p.repetition_penalty))
    fr = float(np.float32(p.frequency_penalty))
    pr = float(np.float32(p.presence_penalty))
    touched = sorted(set(int(t) for t in prompt) | set(int(t) for t in output))
    for v in touched:                      # only ids with cnt_v > 0 or inP_v change
        j = v - vocab_offset
        if not (0 <= j < n):
            continue
        c = int(cnt[v])
        y = float(z[j])
        if mode == PEN_OPENAI_CTRL:
            if r != 1.0:
                y = float(f32(y / r)) if y > 0 else float(f32(y * r))
            if c > 0:
                y = float(f32(y - float(f32(fr * c))))
                y = float(f32(y - pr))
        elif mode == PEN_LINEAR:
            y = float(f32(y - float(f32(fr * c))))
            y = float(f32(y - (pr if c > 0 else 0.0)))
            y = float(f32(y - r))  # here c>0 or inP holds
        else:
            raise ValueError(mode)
        z[j] = np.float32(y)
    return z


# --------------------------------------------------------------------------- filters
def order_pi(zp: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Step 5: pi = all v with w_v > 0 sorted by (z'_v desc, v asc)  (stable lexsort)."""
    ids = np.nonzero(w > 0)[0]
    keys = zp[ids]
    o = np.lexsort((ids, -keys))
    return ids[o]


def top_k_set(pi: np.ndarray, k: int, V: int) -> np.ndarray:
    """Step 6: K1 = pi[0:k] if 1 <= k < V else pi  (strict k, lowest id wins ties)."""
    if 1 <= k < V:
        return pi[:k]
    return pi


def top_p_set(K1: np.ndarray, w: np.ndarray, p: float):
    """Step 7a: smallest prefix of K1 (pi order) whose cumulative weight >= p * W1,
    W1 = sum_{K1} w (top-p on the renormalised post-top-k distribution; R7, R8).
    Returns (K2, j, c, W1) with j the 0-based index of the last kept element."""
    if not (p < 1.0):
        return K1, len(K1) - 1, None, float(np.sum(w[K1]))
    W1 = float(np.sum(w[K1]))
    c = np.cumsum(w[K1])           # sequential float64 running sum, pi order
    target = p * W1
    hit = np.nonzero(c >= target)[0]
    j = int(hit[0]) if len(hit) else len(K1) - 1
    return K1[:j + 1], j, c, W1


def min_p_set(K2: np.ndarray, w: np.ndarray, min_p: float) -> np.ndarray:
    """Step 7b: K3 = {v in K2 : w_v >= min_p}; w_max = 1 so this is p_v >= min_p * p_max
    (R6).  The max always survives."""
    if not (min_p > 0.0):
        return K2
    return K2[w[K2] >= min_p]


def draw_from(K3: np.ndarray, w: np.ndarray, u: float):
    """Step 8: walk K3 in ascending token id; token = first v with cumulative C_v > u*W
    (strict '>' so zero-weight ids are never chosen; R10).
    Returns (token, W, C_tok, C_prev)."""
    ids = np.sort(K3)
    ws = w[ids]
    W = float(np.sum(ws))
    C = np.cumsum(ws)
    target = u * W
    hit = np.nonzero(C > target)[0]
    i = int(hit[0]) if len(hit) else len(ids) - 1
    prev = float(C[i - 1]) if i > 0 else 0.0
    return int(ids[i]), W, float(C[i]), prev


# --------------------------------------------------------------------------- one row
def sample_row(raw_row, dtype: str, prompt, output, p: Params, step: int,
               mode: int = PEN_OPENAI_CTRL, u: float | None = None,
               want_q: bool = False) -> RowResult:
    """The whole chain for one request, float64."""
    x = decode_logits(raw_row, dtype)
    V = len(x)
    if np.any(np.isnan(x)) or np.any(np.isposinf(x)):
        return RowResult(-1, float("nan"), float("nan"), ROW_NONFINITE, False, False)
    zp = apply_penalties(x.astype(np.float32), prompt, output, p, mode).astype(np.float64)
    greedy = bool(np.float32(p.temperature) < np.float32(GREEDY_EPS))  # R5 (compared in binary32)
    tau = 1.0 if greedy else float(np.float32(p.temperature))
    finite = zp > -np.inf
    if not np.any(finite):
        return RowResult(-1, float("nan"), float("nan"), ROW_ALL_NEG_INF, False, greedy)
    M = float(np.max(zp))                                    # step 4
    w = np.zeros(V)
    w[finite] = np.exp((zp[finite] - M) / tau)
    S = float(np.sum(w))
    pi = order_pi(zp, w)
    if len(pi) == 0:
        return RowResult(-1, float("nan"), float("nan"), ROW_ALL_NEG_INF, False, greedy)
    if u is None:
        u = philox_uniform(p.seed, p.request_id, step)
    flags = {}
    if greedy:
        tok = int(pi[0])                                     # lowest-index argmax (R5, R9)
        lp = (zp[tok] - M) / tau - math.log(S)
        res = RowResult(tok, lp, 0.0, ROW_OK, False, True, M, S, u, np.array([tok]))
        if want_q:
            q = np.zeros(V)
            q[tok] = 1.0
            res.q = q
        return res
    K1 = top_k_set(pi, int(p.top_k), V)
    K2, j, c, W1 = top_p_set(K1, w, float(np.float32(p.top_p)))
    mp = float(np.float32(p.min_p))
    K3 = min_p_set(K2, w, mp)
    tok, W, Ct, Cp = draw_from(K3, w, u)
    lp = (zp[tok] - M) / tau - math.log(S)                   # step 8 / R12
    flp = math.log(w[tok] / W)
    # step 10: boundary flags that excuse a token mismatch, at two bands
    pf = float(np.float32(p.top_p))

    def boundary_flags(eps):
        fl = {}
        if pf < 1.0 and c is not None:
            tgt = pf * W1
            fl["top_p"] = bool(abs(c[j] - tgt) <= eps * W1 or (j > 0 and abs(c[j - 1] - tgt) <= eps * W1))
        if mp > 0.0:
            fl["min_p"] = bool(np.any(np.abs(w[K2] - mp) <= eps))
        tgt = u * W
        fl["draw"] = bool(abs(Ct - tgt) <= eps * W or abs(Cp - tgt) <= eps * W)
        return fl

    flags = boundary_flags(FLAG_EPS_GPU)
    flags6 = boundary_flags(FLAG_EPS)
    res = RowResult(tok, lp, flp, ROW_OK, any(flags.values()), False, M, S, u, np.sort(K3), flags=flags,
                    flagged6=any(flags6.values()), flags6=flags6)
    if want_q:
        q = np.zeros(V)
        q[K3] = w[K3] / W
        res.q = q
    return res


def sample_batch(raw, dtype, prompts, outputs, params, step, mode=PEN_OPENAI_CTRL, want_q=False):
    """Row-by-row loop over a [B x V] batch (no batching tricks: obviously correct)."""
    return [sample_row(raw[b], dtype, prompts[b], outputs[b], params[b], step, mode, want_q=want_q)
            for b in range(len(params))]

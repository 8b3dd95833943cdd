"""Pins for the float64 CPU oracle (oracle/) — each against something other than itself.

Pins used:
  * Random123 known-answer vectors for Philox4x32-10 (tests/golden/philox_kat.txt)
  * SPEC.md hand-computed examples (tests/golden/spec_examples.txt)
  * closed forms: softmax of [0, ln 3], uniform rows, torch.log_softmax(float64)
  * library routines: numpy.argmax (first-occurrence tie-break), torch.topk on tie-free rows,
    numpy float32 IEEE arithmetic for the binary32 penalty emulation
  * brute force on tiny vocabularies with an independent O(V^2) rank formulation
  * chi-squared of >= 1e5 draws against the closed-form filtered softmax
"""
import math
import os

import numpy as np
import pytest

from oracle import Params, sample_row, apply_penalties, draw_from, philox4x32_10, uniform
from oracle.sampler_ref import PEN_LINEAR, PEN_OPENAI_CTRL, ROW_NONFINITE, ROW_ALL_NEG_INF, ROW_OK

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _row(z, **kw):
    return np.asarray(z, dtype=np.float32)


def run(z, p, prompt=(), output=(), step=0, u=None, mode=PEN_OPENAI_CTRL):
    return sample_row(np.asarray(z, dtype=np.float32), "f32", list(prompt), list(output), p, step,
                      mode=mode, u=u, want_q=True)


# ----------------------------------------------------------------------------- RNG
def test_philox_known_answers():
    n = 0
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert philox4x32_10(w[0:4], w[4:6]) == tuple(w[6:10])
        n += 1
    assert n == 3


def test_uniform_range_and_determinism():
    us = [uniform(1234, r, 7) for r in range(2000)]
    assert all(0.0 <= x < 1.0 for x in us)
    assert uniform(1234, 5, 7) == uniform(1234, 5, 7)          # SPEC S:235 determinism
    assert uniform(1234, 5, 7) != uniform(1234, 5, 8)
    assert uniform(1234, 5, 7) != uniform(1235, 5, 7)
    # uniformity (KS against U[0,1))
    from scipy.stats import kstest
    assert kstest(us, "uniform").pvalue > 1e-4
    # 53-bit construction: u * 2^53 is an integer
    x = uniform(99, 1, 1) * 2.0 ** 53
    assert x == int(x)


# ----------------------------------------------------------------------------- penalties
def test_penalty_spec_hand_values():
    # alpha_freq=1, f=2, z=1 -> -1 (paper-literal linear mode)
    p = Params(frequency_penalty=1.0, presence_penalty=0.0, repetition_penalty=0.0)
    z = apply_penalties(np.array([0.0, 1.0], np.float32), [], [1, 1], p, PEN_LINEAR)
    assert z[1] == -1.0 and z[0] == 0.0
    # all alphas 0 -> unchanged
    p0 = Params(frequency_penalty=0.0, presence_penalty=0.0, repetition_penalty=0.0)
    zz = np.array([0.37, -2.5, 4.0], np.float32)
    assert np.array_equal(apply_penalties(zz, [0, 1], [2, 2], p0, PEN_LINEAR), zz)
    assert np.array_equal(apply_penalties(zz, [0, 1], [2, 2], Params(), PEN_OPENAI_CTRL), zz)


def test_penalty_ctrl_hand_values():
    p = Params(repetition_penalty=2.0)
    z = apply_penalties(np.array([2.0, -2.0, 0.0, 5.0], np.float32), [0, 1, 2], [], p)
    assert list(z) == [1.0, -4.0, 0.0, 5.0]          # y>0 divides, y<=0 multiplies; 3 untouched
    # frequency/presence on outputs only: z=1, freq=0.5 cnt=3, pres=0.25 -> 1-1.5-0.25
    p = Params(frequency_penalty=0.5, presence_penalty=0.25)
    z = apply_penalties(np.array([1.0, 1.0], np.float32), [1], [0, 0, 0], p)
    assert z[0] == -0.75 and z[1] == 1.0               # prompt-only token: no freq/pres (R2)


def test_penalty_history_prompt_semantics():
    # prompt [3,3,7] -> repetition indicator on {3,7}, frequency 0
    p = Params(repetition_penalty=2.0, frequency_penalty=1.0, presence_penalty=1.0)
    z = np.full(10, 4.0, np.float32)
    out = apply_penalties(z, [3, 3, 7], [], p)
    assert out[3] == 2.0 and out[7] == 2.0
    assert np.all(np.delete(out, [3, 7]) == 4.0)
    # append [5] twice -> count 2
    out = apply_penalties(z, [], [5, 5], Params(frequency_penalty=1.0))
    assert out[5] == 2.0


def test_penalty_binary32_rounding_matches_numpy_ieee():
    """The float64-op-then-round emulation equals numpy's native binary32 arithmetic."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        x = np.float32(rng.normal() * 10)
        r = np.float32(rng.uniform(0.5, 2.0))
        fr = np.float32(rng.uniform(0, 1))
        pr = np.float32(rng.uniform(-1, 1))
        c = int(rng.integers(1, 40))
        p = Params(repetition_penalty=float(r), frequency_penalty=float(fr), presence_penalty=float(pr))
        got = apply_penalties(np.array([x], np.float32), [], [0] * c, p)[0]
        y = (x / r) if x > 0 else (x * r)                  # numpy float32 ops are IEEE binary32
        y = np.float32(y - np.float32(fr * np.float32(c)))
        y = np.float32(y - pr)
        assert got == y
        gl = apply_penalties(np.array([x], np.float32), [], [0] * c, p, PEN_LINEAR)[0]
        yl = np.float32(np.float32(np.float32(x - np.float32(fr * np.float32(c))) - pr) - r)
        assert gl == yl


# ----------------------------------------------------------------------------- softmax / logprob
def test_softmax_closed_forms():
    r = run([0.0, math.log(3.0)], Params(temperature=1.0))
    assert np.allclose(r.q, [0.25, 0.75], rtol=0, atol=1e-7)       # SPEC S:215 (ln 3 rounded to fp32)
    V = 7
    r = run(np.zeros(V), Params(temperature=1.0))
    assert np.allclose(r.q, 1.0 / V, atol=1e-15)
    assert abs(r.logprob + math.log(V)) < 1e-15


def test_logprob_matches_torch_log_softmax():
    import torch
    rng = np.random.default_rng(1)
    for t in (0.5, 0.7, 1.0, 1.7):
        z = (rng.normal(size=300) * 3).astype(np.float32)
        p = Params(temperature=t, seed=3, request_id=9)
        r = run(z, p)
        zt = torch.tensor(z.astype(np.float64)) / float(np.float32(t))
        ref = torch.log_softmax(zt, dim=0)[r.token].item()
        assert abs(r.logprob - ref) < 1e-12


# ----------------------------------------------------------------------------- greedy / top-k
def test_greedy_is_numpy_argmax_first_occurrence():
    rng = np.random.default_rng(2)
    for i in range(200):
        z = rng.integers(-5, 5, size=50).astype(np.float32)    # many exact ties
        zp = apply_penalties(z, [], [], Params())
        r = run(z, Params(temperature=0.0, seed=i))
        assert r.token == int(np.argmax(zp))
        r1 = run(z, Params(temperature=0.8, top_k=1, seed=i, request_id=i))
        assert r1.token == int(np.argmax(zp))                  # top_k=1 == greedy
    # tau < 1e-5 is greedy; logprob uses tau_eff = 1
    z = np.array([1.0, 3.0, 3.0, 0.0], np.float32)
    r = run(z, Params(temperature=5e-6))
    assert r.token == 1 and r.greedy
    assert abs(r.logprob - (0 - math.log(np.exp(z.astype(np.float64) - 3).sum()))) < 1e-15


def test_top_k_matches_torch_topk_on_tie_free_rows():
    import torch
    rng = np.random.default_rng(3)
    for _ in range(50):
        V = 200
        z = rng.permutation(V).astype(np.float32) * np.float32(0.01)
        k = int(rng.integers(1, V))
        r = run(z, Params(temperature=1.0, top_k=k, seed=1))
        ref = set(torch.topk(torch.tensor(z.astype(np.float64)), k).indices.tolist())
        assert set(np.nonzero(r.q)[0].tolist()) == ref


# ----------------------------------------------------------------------------- spec filter examples
def test_spec_filter_examples():
    lp = np.log(np.array([0.5, 0.3, 0.2]))
    r = run(lp, Params(temperature=1.0, top_p=0.7))
    assert np.allclose(r.q, [0.625, 0.375, 0.0], atol=1e-7)           # SPEC S:224 (fp32 logits)
    z = np.random.default_rng(4).normal(size=12).astype(np.float32)
    r = run(z, Params(temperature=1.0, top_k=12, top_p=1.0, min_p=0.0))
    e = np.exp(z.astype(np.float64) - z.max())
    assert np.allclose(r.q, e / e.sum(), atol=1e-15)                   # SPEC S:225 identity
    r = run(np.log(np.array([0.6, 0.3, 0.1])), Params(temperature=1.0, min_p=0.2))
    assert np.allclose(r.q, [2 / 3, 1 / 3, 0.0], atol=1e-7)            # min-p hand example


def test_spec_draw_examples():
    w = np.array([0.25, 0.75])
    tok, W, _, _ = draw_from(np.array([0, 1]), w, 0.5)
    assert tok == 1
    for u in (0.0, 0.3, 0.999999):
        w1 = np.zeros(6); w1[3] = 1.0
        assert draw_from(np.array([3]), w1, u)[0] == 3
    r = run([0.0, math.log(3.0)], Params(temperature=1.0), u=0.5)
    assert r.token == 1
    r = run([0.0, math.log(3.0)], Params(temperature=1.0), u=0.2)
    assert r.token == 0


# ----------------------------------------------------------------------------- brute force, tiny V
def brute_q(zp, p):
    """Independent O(V^2) formulation of K3 (no sorting): rank by pairwise comparison."""
    V = len(zp)
    tau = 1.0 if np.float32(p.temperature) < np.float32(1e-5) else float(np.float32(p.temperature))
    M = max(zp)
    w = [math.exp((float(z) - M) / tau) for z in zp]
    ahead = lambda a, b: zp[b] > zp[a] or (zp[b] == zp[a] and b < a)   # b precedes a in pi
    rank = [sum(1 for b in range(V) if ahead(a, b)) for a in range(V)]
    k = p.top_k
    K1 = [a for a in range(V) if (rank[a] < k if 1 <= k < V else True)]
    if np.float32(p.temperature) < np.float32(1e-5):
        K3 = [a for a in range(V) if rank[a] == 0]
    else:
        W1 = sum(w[a] for a in K1)
        pp = float(np.float32(p.top_p))
        if pp < 1.0:
            # kept iff the mass strictly ahead of it (within K1) is < p*W1
            K2 = [a for a in K1 if sum(w[b] for b in K1 if ahead(a, b)) < pp * W1]
        else:
            K2 = K1
        mp = float(np.float32(p.min_p))
        K3 = [a for a in K2 if w[a] >= mp] if mp > 0 else K2
    W = sum(w[a] for a in K3)
    q = np.zeros(V)
    for a in K3:
        q[a] = w[a] / W
    return q


def test_brute_force_tiny_vocab():
    rng = np.random.default_rng(5)
    for i in range(400):
        V = int(rng.integers(1, 9))
        z = np.round(rng.normal(size=V) * 2, 1).astype(np.float32)    # ties possible
        p = Params(temperature=float(rng.choice([0.0, 0.5, 1.0, 2.0])),
                   top_k=int(rng.integers(0, V + 2)), top_p=float(rng.choice([1.0, 0.3, 0.6, 0.9])),
                   min_p=float(rng.choice([0.0, 0.1, 0.5])), seed=i, request_id=i)
        r = run(z, p)
        assert r.status == ROW_OK
        qb = brute_q(apply_penalties(z, [], [], Params()).astype(np.float64).tolist(), p)
        if r.flagged:
            continue
        assert np.allclose(r.q, qb, atol=1e-12), (z, p, r.q, qb)
        assert r.q[r.token] > 0
        assert abs(r.filtered_logprob - math.log(r.q[r.token])) < 1e-12 or r.greedy


# ----------------------------------------------------------------------------- chi-squared
def test_chi_squared_draws_vs_closed_form():
    from scipy.stats import chisquare
    rng = np.random.default_rng(6)
    V = 48
    z = (rng.normal(size=V) * 1.5).astype(np.float32)
    for p in (Params(temperature=1.0), Params(temperature=0.8, top_k=20, top_p=0.9, min_p=0.02)):
        r0 = run(z, p)
        q = brute_q(z.astype(np.float64).tolist(), p)
        assert np.allclose(r0.q, q, atol=1e-12)
        K3 = np.nonzero(q > 0)[0]
        w = np.zeros(V); w[K3] = q[K3]
        n = 100_000
        counts = np.zeros(V)
        for req in range(n):
            tok = draw_from(K3, w, uniform(77, req, 3))[0]
            counts[tok] += 1
        assert chisquare(counts[K3], q[K3] * n).pvalue > 1e-4
    # end-to-end through sample_row (request ids vary; fewer draws)
    p = Params(temperature=0.9, top_k=10, seed=5)
    q = brute_q(z.astype(np.float64).tolist(), p)
    counts = np.zeros(V)
    n = 20_000
    for req in range(n):
        p.request_id = req
        counts[run(z, p).token] += 1
    K3 = np.nonzero(q > 0)[0]
    assert chisquare(counts[K3], q[K3] * n).pvalue > 1e-4


# ----------------------------------------------------------------------------- status / invariants
def test_row_status():
    assert run([0.0, float("nan")], Params()).status == ROW_NONFINITE
    assert run([0.0, float("inf")], Params()).status == ROW_NONFINITE
    assert run([-np.inf, -np.inf], Params()).status == ROW_ALL_NEG_INF
    r = run([-np.inf, 1.0, -np.inf], Params(temperature=1.0))
    assert r.status == ROW_OK and r.token == 1 and abs(r.logprob) < 1e-15


def test_invariants_random_rows():
    rng = np.random.default_rng(8)
    for i in range(100):
        V = int(rng.integers(2, 400))
        z = (rng.normal(size=V) * 3).astype(np.float32)
        p = Params(temperature=float(rng.choice([0.3, 1.0])), top_k=int(rng.integers(0, V)),
                   top_p=float(rng.choice([1.0, 0.9])), min_p=float(rng.choice([0.0, 0.05])),
                   repetition_penalty=1.2, frequency_penalty=0.3, presence_penalty=0.1, seed=i)
        hist = rng.integers(0, V, size=20).tolist()
        r = run(z, p, prompt=hist[:10], output=hist[10:])
        assert abs(r.q.sum() - 1.0) < 1e-12
        assert r.q[r.token] > 0 and r.logprob <= 1e-15
        assert set(np.nonzero(r.q)[0]) == set(r.kept.tolist())


def test_exact_boundaries_ge_semantics():
    """Exactly representable boundaries: top-p stops at cumulative == p*W1 (>=, R8);
    min-p keeps w == min_p (>=, R6); draw uses strict > (R10)."""
    z = np.zeros(4, np.float32)                       # w = 1 each, W1 = 4
    r = run(z, Params(temperature=1.0, top_p=0.5))
    assert list(r.kept) == [0, 1]                     # c = 1, 2 >= 2.0 -> stop at j=1
    r = run(z, Params(temperature=1.0, min_p=1.0))
    assert list(r.kept) == [0, 1, 2, 3]
    w = np.ones(4)
    assert draw_from(np.arange(4), w, 0.25)[0] == 1   # C = 1,2,.. ; u*W = 1.0; first C > 1 -> id 1
    assert draw_from(np.arange(4), w, 0.0)[0] == 0


# ----------------------------------------------------------------------------- pins added in round 2
def _kat_rows():
    rows = []
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        rows.append([int(x, 16) for x in line.split()])
    return rows


def test_uniform_word_and_counter_mapping_from_kat():
    """DESIGN.md R11 / SURVEY §8c-9: key = (seed_lo, seed_hi), counter = (step_lo, step_hi,
    request_lo, request_hi), u = ((x1 << 32 | x0) >> 11) * 2^-53.  Each published Random123 vector
    is re-read as a (seed, request, step) triple, so a swapped word, counter slot or shift in
    uniform() fails here (the KAT test above only pins philox4x32_10 itself)."""
    for w in _kat_rows():
        c0, c1, c2, c3, k0, k1, x0, x1 = w[:8]
        seed = (k1 << 32) | k0
        step = (c1 << 32) | c0
        req = (c3 << 32) | c2
        expect = (((x1 << 32) | x0) >> 11) * 2.0 ** -53
        assert uniform(seed, req, step) == expect
    # the first vector written out: all-zero key and counter -> x0 = 0x6627e8d5, x1 = 0xe169c58d
    assert uniform(0, 0, 0) == ((0xE169C58D << 32 | 0x6627E8D5) >> 11) * 2.0 ** -53


def test_decode_bf16_all_bit_patterns_match_torch():
    """Step 1 for dtype 'bf16' against torch's bfloat16 -> float64 conversion on
    every one of the 65536 bit patterns (NaN patterns compared as NaN)."""
    import torch
    from oracle import decode_logits
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = decode_logits(bits, "bf16")
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan], ref[~nan])
    # signed zeros and infinities keep their sign
    assert np.array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))


def _p(**kw):
    return Params(**kw)


def test_flags_top_p_boundary_both_bands():
    """SURVEY §8c-10 top-p flag: |c_j - p*W1| <= eps*W1 (or the same for c_{j-1}).  2048 equal
    logits give w = 1 exactly, so W1 = 2048 and c_j = j + 1 exactly; p = 2^-11 + m*2^-34 is exact in
    binary32 and puts p*W1 exactly m*2^-23 above c_0 = 1: the gap is known to the last bit."""
    from oracle.sampler_ref import FLAG_EPS, FLAG_EPS_GPU
    z = np.zeros(2048, np.float32)
    for m, f6, fg in ((1, True, True), (4000, True, False), (20000, False, False)):
        p = 2.0 ** -11 + m * 2.0 ** -34
        assert float(np.float32(p)) == p
        gap = m * 2.0 ** -23 / 2048.0                   # |c_0 - p*W1| / W1
        assert (gap <= FLAG_EPS) == f6 and (gap <= FLAG_EPS_GPU) == fg
        r = run(z, _p(temperature=1.0, top_p=p, seed=3), u=0.7)
        assert list(r.kept) == [0, 1]                    # c_0 = 1 < p*W1 <= c_1 = 2
        assert r.flags6["top_p"] == f6 and r.flags["top_p"] == fg, (m, r.flags6, r.flags)
        assert r.flagged6 == f6 and r.flagged == fg      # u = 0.7 is far from the draw boundary


def test_flags_min_p_boundary_both_bands():
    """min-p flag: some kept w_v within eps of min_p (absolute: w_max = 1).  The element's weight is
    w = e^-14 (logit -14 exact in binary32, max 0); min_p is a binary32 a known distance from it
    (near 2^-20 the binary32 spacing is 2^-44, far below both bands)."""
    from oracle.sampler_ref import FLAG_EPS, FLAG_EPS_GPU
    w1 = math.exp(-14.0)
    z = np.array([0.0, -14.0, -30.0], np.float32)
    for dist, f6, fg in ((4e-11, True, True), (-4e-11, True, True), (5e-7, True, False), (2e-6, False, False)):
        mp = float(np.float32(w1 + dist))
        d = abs(w1 - mp)
        assert abs(d - abs(dist)) < 1e-13
        r = run(z, _p(temperature=1.0, min_p=mp, seed=1), u=0.3)
        assert r.flags6["min_p"] == f6 and r.flags["min_p"] == fg, (dist, r.flags6, r.flags)
        assert (1 in r.kept.tolist()) == (w1 >= mp)
        assert 2 not in r.kept.tolist()                  # w = e^-30 < min_p


def test_flags_draw_boundary_both_bands():
    """draw flag: |C_tok - u*W| or |C_prev - u*W| <= eps*W, with u passed in explicitly."""
    z = np.array([0.0, 0.0, 0.0, 0.0], np.float32)     # w = 1 each, W = 4, C = 1, 2, 3, 4
    for du, f6, fg in ((2e-7, True, False), (2e-11, True, True), (-2e-11, True, True), (1e-3, False, False)):
        u = 0.5 + du                                   # u*W = 2 + 4*du: next to C = 2
        r = run(z, _p(temperature=1.0, seed=1), u=u)
        assert r.flags6["draw"] == f6 and r.flags["draw"] == fg, (du, r.flags6, r.flags)
        assert r.token == (2 if du > 0 else 1)
        assert r.flagged == fg and r.flagged6 == f6

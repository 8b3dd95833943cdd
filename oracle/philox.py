"""Philox4x32-10 counter-based generator — ORACLE SIDE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import anything under oracle/.  The CUDA path has its own, independent Philox
(paper_2506_22033_b200/csrc/philox.cuh); the two share no code.

Why Philox: the paper's draw is y ~ Categorical(p) (§2.1 step (3));
SPEC.md S:230 fixes a counter-based deterministic generator so that the
reference and the optimised sampler draw the *same* uniform; the north star keys
it by (seed, request, step).  DESIGN.md reading R11 / SURVEY §8c-9:

    key     = (seed_lo, seed_hi)
    counter = (step_lo, step_hi, request_lo, request_hi)
    u       = ((x1 << 32 | x0) >> 11) * 2**-53        in [0, 1)

Pinned by the Random123 known-answer vectors in tests/golden/philox_kat.txt.
Pure-Python integer arithmetic: slow and obviously correct.
"""

MASK32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85


def _mulhilo(a, b):
    p = (a * b) & 0xFFFFFFFFFFFFFFFF
    return p >> 32, p & MASK32


def philox4x32_10(counter, key):
    """Return the 4 output words of Philox4x32 with 10 rounds.

    counter: 4 uint32 words (c0..c3); key: 2 uint32 words (k0, k1).
    Round: (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)),
    key bumped by the Weyl constants (W0, W1) between rounds (Salmon et al. 2011).
    """
    c0, c1, c2, c3 = (int(x) & MASK32 for x in counter)
    k0, k1 = (int(x) & MASK32 for x in key)
    for r in range(10):
        if r:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        hi0, lo0 = _mulhilo(PHILOX_M0, c0)
        hi1, lo1 = _mulhilo(PHILOX_M1, c2)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def uniform(seed, request_id, step):
    """u in [0,1) for one row: DESIGN.md reading R11."""
    seed &= 0xFFFFFFFFFFFFFFFF
    request_id &= 0xFFFFFFFFFFFFFFFF
    step &= 0xFFFFFFFFFFFFFFFF
    key = (seed & MASK32, seed >> 32)
    ctr = (step & MASK32, step >> 32, request_id & MASK32, request_id >> 32)
    x0, x1, _x2, _x3 = philox4x32_10(ctr, key)
    return (((x1 << 32) | x0) >> 11) * (2.0 ** -53)

"""NEXT-3 comparator: the paper's column-wise CPU sampler (baselines/paper_cpu) against the float64
oracle.  It computes in binary32 values with float64 sums (a production CPU sampler, not the
oracle), so tokens must equal the oracle's on every row the oracle does not flag at the north
star's 1e-6 band, and logprobs agree to 1e-4 relative."""
import math

import numpy as np
import pytest

from oracle import sample_row
from tests._helpers import oracle_params
from workloads.synth import RowParams, Workload, gen_logits, make_workload, random_params


def _check(wl, step=0, append_steps=1):
    from baselines.paper_cpu import PaperCpuSampler
    s = PaperCpuSampler(wl.V, wl.B, max_output=4096, threads=4)
    for b in range(wl.B):
        s.set_params(b, wl.params[b])
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    outputs = [list(o) for o in wl.outputs]
    mism = 0
    for st in range(step, step + append_steps):
        tok, lp = s.step(wl.raw, st, append=True)
        for b in range(wl.B):
            o = sample_row(wl.raw[b], wl.dtype, wl.prompts[b], outputs[b], oracle_params(wl.params[b]), st)
            if o.token != tok[b]:
                mism += 1
                assert o.flagged6, (st, b, int(tok[b]), o.token)
            else:
                assert math.isclose(math.exp(lp[b]), math.exp(o.logprob), rel_tol=1e-4, abs_tol=1e-7), (b, lp[b], o.logprob)
            outputs[b].append(int(tok[b]))
    return mism


@pytest.mark.parametrize("cfg", ["c3", "c2", "c4", "c1"])
def test_paper_cpu_sampler_matches_oracle(cfg):
    wl = make_workload(cfg, B=20, V=12000 if cfg != "c1" else 32000)
    _check(wl, step=0, append_steps=3)


def test_paper_cpu_sampler_random_params():
    rng = np.random.default_rng(3)
    B, V = 24, 5000
    raw = gen_logits(rng, B, V, "bf16")
    prompts, outputs = [], []
    for b in range(B):
        n = int(rng.integers(0, 60))
        t = rng.integers(0, V, size=n).tolist()
        prompts.append(t[: n // 2])
        outputs.append(t[n // 2:])
    params = [random_params(rng, b, V) for b in range(B)]
    _check(Workload("rand", B, V, "bf16", raw, prompts, outputs, params), step=5, append_steps=2)

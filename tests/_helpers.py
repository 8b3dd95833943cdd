"""Shared test helpers: build the same seeded workload for the oracle and the CUDA path and
compare them with the north-star parity rule:
  * greedy / argmax ids bit-exact
  * stochastic rows: exp(logprob) and q within 1e-5 relative or 1e-6 absolute
  * token ids identical except in rows the oracle flags (a cutoff or u within FLAG_EPS_GPU = 1e-10 of a
    boundary, R16; rows within the north star's 1e-6 are counted as flagged6)
"""
from __future__ import annotations

import math

import numpy as np

from oracle import Params, sample_row
from workloads.synth import Workload, device_logits  # noqa: F401 (re-export)

REL, ABS = 1e-5, 1e-6


def oracle_params(p) -> Params:
    return Params(**{k: getattr(p, k) for k in Params.__dataclass_fields__})


def oracle_run(wl: Workload, step: int, want_q=False, mode=0, rows=None):
    rows = range(wl.B) if rows is None else rows
    return {b: sample_row(wl.raw[b], wl.dtype, wl.prompts[b], wl.outputs[b], oracle_params(wl.params[b]), step,
                          mode=mode, want_q=want_q) for b in rows}


def make_sampler(wl: Workload, max_history=None, max_top_k=128, mode=0, max_batch=None, **kw):
    from paper_2506_22033_b200 import Sampler
    L = max_history or max(64, max((len(p) + len(o) for p, o in zip(wl.prompts, wl.outputs)), default=0) + 64)
    s = Sampler(wl.V, max_batch or wl.B, max_history=L, max_top_k=max_top_k, dtype=wl.dtype, penalty_mode=mode,
                **kw)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        if wl.prompts[b] or wl.outputs[b]:
            s.set_history(b, wl.prompts[b], wl.outputs[b])
    return s


def close(a, b):
    return abs(a - b) <= max(REL * abs(b), ABS)


def assert_parity(wl: Workload, out: dict, orc: dict, q=None, stats=None):
    """out: dict of torch tensors from Sampler.sample/debug_distribution; orc: {row: RowResult}."""
    tok = out["tokens"].cpu().numpy()
    lp = out["logprobs"].cpu().numpy().astype(np.float64)
    st = out["status"].cpu().numpy() if "status" in out and out["status"] is not None else None
    flp = out["filtered_logprobs"].cpu().numpy().astype(np.float64) if out.get("filtered_logprobs") is not None \
        else None
    qn = q.cpu().numpy() if q is not None else None
    nflag = nmis = nflag6 = 0
    for b, o in orc.items():
        if o.status != 0:
            assert tok[b] == -1, (b, tok[b])
            if st is not None:
                assert st[b] == o.status, (b, st[b], o.status)
            continue
        if st is not None:
            assert st[b] == 0, (b, st[b])
        if o.greedy:
            assert tok[b] == o.token, f"row {b}: greedy token {tok[b]} != oracle {o.token}"
        elif tok[b] != o.token:
            assert o.flagged, f"row {b}: token {tok[b]} != oracle {o.token} and row not flagged ({o.flags})"
            nmis += 1
        nflag += int(o.flagged)
        nflag6 += int(o.flagged6)
        if tok[b] == o.token:
            assert close(math.exp(lp[b]), math.exp(o.logprob)), (b, lp[b], o.logprob)
            if flp is not None and not o.flagged:
                assert close(math.exp(flp[b]), math.exp(o.filtered_logprob)), (b, flp[b], o.filtered_logprob)
        if qn is not None and o.q is not None and not o.flagged:
            d = np.abs(qn[b].astype(np.float64) - o.q)
            tol = np.maximum(REL * o.q, ABS)
            bad = np.nonzero(d > tol)[0]
            assert len(bad) == 0, f"row {b}: q mismatch at {bad[:10]} gpu={qn[b][bad[:5]]} orc={o.q[bad[:5]]}"
    if stats is not None:
        stats["rows"] = stats.get("rows", 0) + len(orc)
        stats["flagged"] = stats.get("flagged", 0) + nflag
        stats["mismatch"] = stats.get("mismatch", 0) + nmis
        stats["flagged6"] = stats.get("flagged6", 0) + nflag6
    return nflag, nmis

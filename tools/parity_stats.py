"""North-star parity statistics: the CUDA path against the float64 oracle over >= 1e5 rows of the
c1-c4 shapes (BASELINE.json configs[0..3]), many steps / request ids / logits draws.

    python tools/parity_stats.py [--rows 100000] [--out profiles/parity_r02.json]

For every row: token equality, exp(logprob) and exp(filtered logprob) within 1e-5 rel / 1e-6 abs
(north star), and the oracle's boundary flags at the excuse band (1e-9, R16) and at the
north star's literal 1e-6.  A token mismatch on an unflagged row is a parity failure.  The oracle
runs in one process per host core.  Writes one JSON summary (per config and total).
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import sample_row  # noqa: E402
from oracle.sampler_ref import FLAG_EPS, FLAG_EPS_GPU  # noqa: E402
from tests._helpers import make_sampler, oracle_params  # noqa: E402
from workloads.synth import device_logits, make_workload  # noqa: E402

REL, ABS = 1e-5, 1e-6
_JOB = None


def _orc(args):
    rows, step = args
    wl = _JOB
    out = []
    for b in rows:
        o = sample_row(wl.raw[b], wl.dtype, wl.prompts[b], wl.outputs[b], oracle_params(wl.params[b]), step)
        out.append((b, o.token, o.logprob, o.filtered_logprob, o.status, o.flagged, o.flagged6, o.greedy,
                    {k: v for k, v in o.flags.items() if v}))
    return out


def close(a, b):
    return abs(a - b) <= max(REL * abs(b), ABS)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r02.json"))
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--sharded", type=int, default=0,
                    help="G > 0: the vocab-sharded path (G slices in one process: local pass, merge, resolve rounds)")
    a = ap.parse_args()
    import torch
    global _JOB
    cfgs = a.configs.split(",")
    # rows per config: equal shares; each (workload draw, step) call samples a whole batch
    share = a.rows // len(cfgs) + 1
    cores = len(os.sched_getaffinity(0))
    summary = {"path": f"vocab-sharded G={a.sharded} (merge + resolve rounds)" if a.sharded else "sampler_sample",
               "rows": 0, "flagged": 0, "flagged6": 0, "mismatch": 0, "unflagged_mismatch": 0,
               "prob_violations": 0, "status_mismatch": 0, "per_config": {}, "cores": cores,
               "band": {"excuse": FLAG_EPS_GPU, "north_star": FLAG_EPS}, "tolerance": {"rel": REL, "abs": ABS}}
    t0 = time.time()
    ctx = mp.get_context("fork")
    for cfg in cfgs:
        st = dict(rows=0, flagged=0, flagged6=0, mismatch=0, unflagged_mismatch=0, prob_violations=0,
                  status_mismatch=0, greedy_rows=0, max_rel_err_p=0.0, draws=0, failures=[])
        draw = 0
        while st["rows"] < share:
            wl = make_workload(cfg, seed_offset=100 + draw, run=draw)
            s = make_sampler(wl) if not a.sharded else None
            x = device_logits(wl)
            steps = max(1, min(8, -(-(share - st["rows"]) // wl.B)))
            _JOB = wl
            with ctx.Pool(cores) as pool:
                for step in range(steps):
                    if a.sharded:
                        from tests.test_gpu_resolve import sharded_inprocess
                        out = sharded_inprocess(wl, x, a.sharded, step)[0][0]
                    else:
                        out = s.sample(x, step)
                    torch.cuda.synchronize()
                    tok = out["tokens"].cpu().numpy()
                    lp = out["logprobs"].cpu().numpy().astype(np.float64)
                    flp = out["filtered_logprobs"].cpu().numpy().astype(np.float64)
                    sts = out["status"].cpu().numpy()
                    rows = list(range(wl.B))
                    res = [r for part in pool.map(_orc, [(rows[i::cores], step) for i in range(cores)]) for r in part]
                    for (b, otok, olp, oflp, ost, fl, fl6, greedy, flags) in res:
                        st["rows"] += 1
                        if ost != 0 or sts[b] != 0:
                            if ost != sts[b] or (ost != 0 and tok[b] != -1):
                                st["status_mismatch"] += 1
                            continue
                        st["greedy_rows"] += int(greedy)
                        st["flagged"] += int(fl)
                        st["flagged6"] += int(fl6)
                        if tok[b] != otok:
                            st["mismatch"] += 1
                            if greedy or not fl:
                                st["unflagged_mismatch"] += 1
                                if len(st["failures"]) < 10:
                                    st["failures"].append(dict(draw=draw, step=step, row=b, gpu=int(tok[b]),
                                                               oracle=int(otok)))
                        else:
                            pg, po = math.exp(lp[b]), math.exp(olp)
                            e = abs(pg - po) / max(po, 1e-300)
                            st["max_rel_err_p"] = max(st["max_rel_err_p"], e)
                            bad = not close(pg, po)
                            if not greedy and not fl:
                                bad |= not close(math.exp(flp[b]), math.exp(oflp))
                            st["prob_violations"] += int(bad)
            st["draws"] += 1
            draw += 1
            del s
        summary["per_config"][cfg] = st
        for k in ("rows", "flagged", "flagged6", "mismatch", "unflagged_mismatch", "prob_violations",
                  "status_mismatch"):
            summary[k] += st[k]
        print(cfg, {k: v for k, v in st.items() if k != "failures"}, "elapsed %.0fs" % (time.time() - t0), flush=True)
    summary["flag_frac"] = summary["flagged"] / max(1, summary["rows"])
    summary["flag6_frac"] = summary["flagged6"] / max(1, summary["rows"])
    summary["mismatch_frac"] = summary["mismatch"] / max(1, summary["rows"])
    summary["pass"] = summary["unflagged_mismatch"] == 0 and summary["prob_violations"] == 0 and \
        summary["status_mismatch"] == 0
    summary["wall_s"] = time.time() - t0
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "per_config"}))


if __name__ == "__main__":
    main()

"""Phase timeline of one c3 sampling call (SAMPLER_TRACE=1 build-time-free device timestamps).

Prints, relative to the first phase-A warp start (ns): phase-A warp start / end percentiles and,
for phase B, the per-row timestamp of every traced phase (median / max over rows)."""
import os
import sys

os.environ["SAMPLER_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes

import numpy as np
import torch

from paper_2506_22033_b200 import Sampler
from paper_2506_22033_b200 import sampler as smod
from workloads.synth import device_logits
from workloads.synth import make_workload


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    wl = make_workload(cfg, B=int(os.environ["TRACE_B"]) if os.environ.get("TRACE_B") else None)
    s = Sampler(wl.V, wl.B, max_history=2048, max_top_k=128, dtype=wl.dtype)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    xs = [device_logits(make_workload(cfg, seed_offset=j)) for j in range(5)] if os.environ.get("COLD") else [device_logits(wl)]
    for i in range(5):
        s.sample(xs[i % len(xs)], i)
    torch.cuda.synchronize()
    s.sample(xs[-1 if len(xs) == 1 else 0], 9)
    torch.cuda.synchronize()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    vec = 8 if wl.dtype == "bf16" else 4
    spr = -(-(-(-wl.V // vec)) // 128)
    nA = 64 * (wl.B * spr // int(os.environ.get("TILE_STEPS", "26")) + 1)
    n = nA + 32 * wl.B
    buf = (ctypes.c_uint64 * n)()
    rc = smod._lib.sampler_debug_trace(s.h, buf, n)
    assert rc == 0, rc
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
    A = t[:nA].reshape(-1, 64)
    st, en = A[:, 0], A[:, 7]
    used = st > 0
    t0 = st[used].min()
    pr = lambda v: f"p0={np.percentile(v, 0):8.0f} p50={np.percentile(v, 50):8.0f} p90={np.percentile(v, 90):8.0f} max={v.max():8.0f}"
    print("phaseA start", pr(st[used] - t0))
    sm = A[used, 1]
    print("phaseA CTAs", int(used.sum()), "distinct SMs", len(set(sm.tolist())))
    order = np.argsort(st[used])
    late = (st[used] - t0) > 2000
    print("late CTAs", int(late.sum()), "their SMs", sorted(set(sm[late].tolist()))[:40])
    print("per-CTA (start,end) us of late:", [(round((st[used][i]-t0)/1e3,1), round((en[used][i]-t0)/1e3,1)) for i in np.where(late)[0][:10]])
    print("phaseA end  ", pr(en[used] - t0))
    # (per-warp consumer wait times are no longer recorded: the stamps cost ~0.5 us in the loop)
    print("producer empty-wait ns p50=%.0f max=%.0f ; producer done p50=%.0f" % (np.median(A[used, 9]), A[used, 9].max(), np.median(A[used, 10] - t0)))
    pw = A[used, 8]
    print("penalty warp end", pr(pw[pw > 0] - t0))
    Bt = t[nA:].reshape(wl.B, 32)
    for k in range(32):
        v = Bt[:, k]
        v = v[v > 0]
        if len(v):
            print(f"phaseB[{k:2d}]  ", pr(v - t0), f"rows={len(v)}")


if __name__ == "__main__":
    main()

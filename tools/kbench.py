"""Feature-isolation timing of the sampler kernel (development tool, not the driver bench).

Times sampler.sample on B x V bf16 logits with variants that switch features off, next to
torch reference reductions of the same bytes.  CUDA events, rotating buffers (> L2).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2506_22033_b200 import Sampler, SamplingParams


def timeit(fn, xs, iters=50, warm=5):
    for i in range(warm):
        fn(xs[i % len(xs)], i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(xs[i % len(xs)], i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1000.0  # us


def ktimes(s, fn, xs, iters=30, warm=3):
    """Per-kernel device times (us) via the library's own CUDA events on the launch stream."""
    for i in range(warm):
        fn(xs[i % len(xs)], i)
    s.set_timing(True)
    acc = None
    for i in range(iters):
        fn(xs[i % len(xs)], warm + i)
        t = s.kernel_times_ms()
        acc = t if acc is None else [a + b for a, b in zip(acc, t)]
    s.set_timing(False)
    return [round(a / iters * 1000.0, 2) for a in acc]


def c3_bench(nbuf=5, append=True):
    """The bench.py c3 workload (synthetic logits + histories + params), per-kernel times."""
    from workloads.synth import make_workload
    from workloads.synth import device_logits
    wls = [make_workload("c3", seed_offset=i) for i in range(nbuf)]
    wl = wls[0]
    s = Sampler(wl.V, wl.B, max_history=2048, max_top_k=128, dtype=wl.dtype)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    xs = [device_logits(w) for w in wls]
    out = s._outs(wl.B, None)
    fn = lambda x, i: s.sample(x, i, append=append, out=out)
    return {"c3_total_us": timeit(fn, xs, iters=30), "c3_kernels_us": ktimes(s, fn, xs)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--V", type=int, default=152064)
    ap.add_argument("--nbuf", type=int, default=5)
    args = ap.parse_args()
    B, V = args.B, args.V
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = []
    for i in range(args.nbuf):
        x = (2.0 * torch.randn(B, V, device="cuda", generator=g)).to(torch.bfloat16)
        xs.append(x)
    res = {}
    res["torch_amax_us"] = timeit(lambda x, i: x.amax(dim=1), xs)
    res["torch_copy_us"] = timeit(lambda x, i: x.clone(), xs)
    variants = {
        "greedy": SamplingParams(temperature=0.0),
        "topk40_nopen": SamplingParams(temperature=0.7, top_k=40, top_p=0.9, min_p=0.05),
        "topk40_pen": SamplingParams(temperature=0.7, top_k=40, top_p=0.9, min_p=0.05, repetition_penalty=1.1,
                                     presence_penalty=0.4, frequency_penalty=0.3),
        "topk1": SamplingParams(temperature=0.7, top_k=1),
    }
    rng = np.random.default_rng(0)
    for name, p in variants.items():
        s = Sampler(V, B, max_history=1024, max_top_k=128, dtype="bf16")
        s.set_params(list(range(B)), [p] * B)
        if name.endswith("_pen"):
            for b in range(B):
                s.set_history(b, rng.integers(0, V, 384).tolist(), rng.integers(0, V, 128).tolist())
        out = s._outs(B, None)
        res[name + "_us"] = timeit(lambda x, i: s.sample(x, i, out=out), xs)
        res[name + "_kernels_us"] = ktimes(s, lambda x, i: s.sample(x, i, out=out), xs)
    mb = B * V * 2 / 1e6
    res["MB"] = mb
    res.update(c3_bench())
    print(json.dumps(res))


if __name__ == "__main__":
    main()


def trace(B=32, V=152064, variant="greedy"):
    """SAMPLER_TRACE=1 python -c 'import tools.kbench as k; k.trace()'"""
    import ctypes
    from paper_2506_22033_b200.sampler import lib
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (2.0 * torch.randn(B, V, device="cuda", generator=g)).to(torch.bfloat16)
    p = SamplingParams(temperature=0.0) if variant == "greedy" else SamplingParams(temperature=0.7, top_k=40)
    s = Sampler(V, B, max_history=1024, dtype="bf16")
    s.set_params(list(range(B)), [p] * B)
    for i in range(3):
        s.sample(x, i)
    torch.cuda.synchronize()
    mc = torch.cuda.get_device_properties(0).multi_processor_count * 3
    n = 64 * mc + 32 * B
    buf = (ctypes.c_uint64 * n)()
    assert lib().sampler_debug_trace(s.h, buf, n) == 0
    allt = np.array(buf[:], dtype=np.int64)
    wt = allt[:64 * mc].reshape(-1, 8)
    mt = allt[64 * mc:64 * mc + 32 * B].reshape(-1, 32)
    wt = wt[wt[:, 0] > 0]
    t0 = wt[:, 0].min()
    st_ = wt[:, 0] - t0
    en = wt[:, 7] - t0
    print("warps", len(wt), "start ns: med %d max %d" % (np.median(st_), st_.max()),
          "end ns: min %d med %d p90 %d max %d" % (en.min(), np.median(en), np.percentile(en, 90), en.max()))
    mrel = np.where(mt > 0, mt - t0, -1)
    for c in list(range(0, B, max(1, B // 6))):
        print("merge row", c, [int(v) for v in mrel[c] if v >= 0][:20])
    st = mrel[:, 0]
    print("merge start ns: min %d med %d max %d" % (st.min(), np.median(st), st.max()))

"""HBM bandwidth probes on B200 (development tool): torch read-only reductions and copies over
rotating buffers larger than L2, CUDA events."""
import json
import torch


def t(fn, xs, iters=40):
    for i in range(5):
        fn(xs[i % len(xs)])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(xs[i % len(xs)])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


res = {}
for mb in (78, 256, 1024):
    n = mb * 1024 * 1024 // 2
    nb = max(2, 400 // mb + 1)
    xs = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(nb)]
    by = n * 2
    us = t(lambda x: x.view(-1, 8192).amax(dim=1), xs)
    res[f"amax_{mb}MB"] = (round(us, 2), round(by / us / 1e3, 1))
    us = t(lambda x: x.sum(dtype=torch.float32), xs)
    res[f"sum_{mb}MB"] = (round(us, 2), round(by / us / 1e3, 1))
    ys = [torch.empty_like(x) for x in xs]
    k = [0]
    def cp(x):
        ys[k[0] % len(ys)].copy_(x)
        k[0] += 1
    us = t(cp, xs)
    res[f"copy_{mb}MB(rd+wr)"] = (round(us, 2), round(2 * by / us / 1e3, 1))
    del xs, ys
print(json.dumps(res))

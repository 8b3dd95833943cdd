import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_22033_b200 import Sampler
from workloads.synth import device_logits
from workloads.synth import make_workload
for B in [int(x) for x in os.environ.get("BS", "8,64,256").split(",")]:
    wl = make_workload("c3", B=B)
    s = Sampler(wl.V, wl.B, max_history=2048, max_top_k=128, dtype=wl.dtype)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    x = device_logits(wl)
    for i in range(4):
        t0 = time.time()
        o = s.sample(x, i)
        torch.cuda.synchronize()
        print(B, i, round((time.time() - t0) * 1e3, 2), "ms", o["tokens"][:4].tolist(), flush=True)

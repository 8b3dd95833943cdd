"""A small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): c1 in
full, a c3-shaped batch with in-kernel history append over 3 steps and a CUDA-graph replay, c2
top-p-only rows through the exact cluster kernel, invalid device slots / params, and the
vocab-sharded local pass + merge.  Development tool (tools/sanitize.sh runs it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_22033_b200 import Sampler, params_to_device  # noqa: E402
from tests._helpers import make_sampler  # noqa: E402
from workloads.synth import RowParams, device_logits, make_workload  # noqa: E402

for cfg, B, V in (("c1", None, None), ("c3", 8, 30000), ("c2", 4, 20000), ("c4", 12, 16000)):
    wl = make_workload(cfg, B=B, V=V)
    s = make_sampler(wl)
    x = device_logits(wl)
    for step in range(3):
        s.sample(x, step, append=True)
    torch.cuda.synchronize()
    out = s._outs(wl.B, None)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        s.sample(x, 9, out=out, append=True)
    g.replay()
    torch.cuda.synchronize()
    print(cfg, "ok", out["tokens"].tolist()[:4], flush=True)
# invalid device slots / params
wl = make_workload("c3", B=6, V=9000)
s = make_sampler(wl, max_batch=8)
params = [RowParams(**p.__dict__) for p in wl.params]
params[1].top_p = 0.0
slots = torch.arange(wl.B, dtype=torch.int32, device="cuda")
slots[2] = 99
o = s.sample(device_logits(wl), 0, slots=slots, params=params_to_device(params), append=True)
torch.cuda.synchronize()
print("invalid ok", o["status"].tolist(), flush=True)
# vocab-sharded: 2 slices on one GPU, in-process gather
wl = make_workload("c3", B=6, V=12000)
x = device_logits(wl)
recs, shs = [], []
for lo, hi in ((0, 6000), (6000, 12000)):
    sh = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
    sh.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        sh.set_history(b, wl.prompts[b], wl.outputs[b])
    rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
    sh.sample_local(x[:, lo:hi], rec)
    recs.append(rec)
    shs.append(sh)
o = shs[0].merge(torch.cat(recs), 2, wl.B, 0, append=True)
torch.cuda.synchronize()
print("sharded ok", o["tokens"].tolist(), flush=True)
# NEXT-1: resolve rounds for top-p-only rows (2 slices, in-process gather), with append
wl = make_workload("c2", B=4, V=12000)
x = device_logits(wl)
recs, shs, xs = [], [], []
for g, (lo, hi) in enumerate(((0, 6000), (6000, 12000))):
    sh = Sampler(wl.V, wl.B, max_history=2048, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
    sh.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        sh.set_history(b, wl.prompts[b], wl.outputs[b])
    rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
    sh.sample_local(x[:, lo:hi], rec)
    recs.append(rec)
    shs.append(sh)
    xs.append(x[:, lo:hi])
gat = torch.cat(recs)
outs = [sh.merge(gat, 2, wl.B, 0, append=True) for sh in shs]
pays = [torch.empty(sh.resolve_bytes(wl.B), dtype=torch.uint8, device="cuda") for sh in shs]
act = torch.zeros(1, dtype=torch.int32, device="cuda")
for g, sh in enumerate(shs):
    sh.resolve_round(xs[g], 0, 0, None, 2, g, pays[g], outs[g], append=True, active=act)
for n in range(1, Sampler.resolve_max_rounds() + 1):
    gat = torch.cat(pays)
    for g, sh in enumerate(shs):
        sh.resolve_round(xs[g], 0, n, gat, 2, g, pays[g], outs[g], append=True, active=act)
torch.cuda.synchronize()
print("resolve ok", outs[0]["tokens"].tolist(), outs[0]["status"].tolist(), flush=True)
# NEXT-2: one-shot peer exchange, 2 ranks of one process in lock step
wl = make_workload("c3", B=6, V=12000)
x = device_logits(wl)
shs = []
for g, (lo, hi) in enumerate(((0, 6000), (6000, 12000))):
    sh = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
    sh.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        sh.set_history(b, wl.prompts[b], wl.outputs[b])
    shs.append((sh, lo, hi))
bases = [sh.exchange_init(2, g)[1] for g, (sh, _, _) in enumerate(shs)]
for sh, _, _ in shs:
    sh.exchange_set_peers(bases)
for step in range(2):
    for sh, lo, hi in shs:
        sh.sample_exchange(x[:, lo:hi], step, append=True, phases=1)
    outs = [sh.sample_exchange(x[:, lo:hi], step, append=True, phases=2) for sh, lo, hi in shs]
torch.cuda.synchronize()
print("exchange ok", outs[0]["tokens"].tolist(), flush=True)

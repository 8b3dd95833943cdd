"""Debug: unsharded vs vocab-sharded (in-process gather) logprobs against the oracle."""
import math
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_22033_b200 import Sampler
from paper_2506_22033_b200.distributed import vocab_shard_bounds
from tests._helpers import make_sampler, oracle_run
from workloads.synth import make_workload, device_logits

wl = make_workload("c3", B=32, V=30000)
x = device_logits(wl)
orc = oracle_run(wl, 9)
full = make_sampler(wl)
ref = full.sample(x, 9)
torch.cuda.synchronize()
def err(o):
    lp = o["logprobs"].cpu().numpy().astype(np.float64)
    tok = o["tokens"].cpu().numpy()
    e = [abs(math.exp(lp[b]) / math.exp(orc[b].logprob) - 1) for b in range(wl.B) if tok[b] == orc[b].token]
    return max(e), int(np.argmax(e)), sum(tok[b] != orc[b].token for b in range(wl.B))
print("unsharded", err(ref))
for G in (2, 4, 8):
    shards, recs = [], []
    for r in range(G):
        lo, hi = vocab_shard_bounds(wl.V, G, r)
        sh = Sampler(wl.V, wl.B, max_history=1024, max_top_k=128, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
        sh.set_params(list(range(wl.B)), wl.params)
        for b in range(wl.B):
            sh.set_history(b, wl.prompts[b], wl.outputs[b])
        rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
        sh.sample_local(x[:, lo:hi], rec)
        shards.append(sh); recs.append(rec)
    o = shards[0].merge(torch.cat(recs), G, wl.B, 9)
    torch.cuda.synchronize()
    print("G", G, err(o), [vocab_shard_bounds(wl.V, G, r) for r in range(G)])
    # record headers
    rb = shards[0].record_bytes(wl.B) // wl.B
    for r in range(G):
        h = recs[r].view(wl.B, rb)[0, :48].cpu().numpy()
        m = h[:4].view(np.float32)[0]; s = h[8:16].view(np.float64)[0]; R = h[16:24].view(np.float64)[0]
        print("  rank", r, "row0 m=%.6f s=%.9g R=%.6f n=%d" % (m, s, R, h[24:28].view(np.uint32)[0]))
print("oracle row0 M=%.6f S=%.9g" % (orc[0].M, orc[0].S))

"""Development: the sharded edge rows of tests/test_gpu_resolve.py::test_sharded_edge_rows, printed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_resolve import sharded_inprocess
from tests._helpers import oracle_run, make_sampler
from workloads.synth import RowParams, Workload, device_logits, f32_to_bf16_bits
dtype = sys.argv[1] if len(sys.argv) > 1 else "f32"
B, V = 8, 9000
rng = np.random.default_rng(17)
z = rng.normal(0, 2, size=(B, V)).astype(np.float32)
z[0] = (rng.integers(-50, 50, size=V) * np.float32(1e-41)).astype(np.float32)
z[1] = np.float32(0.0); z[1, ::2] = np.float32(-0.0)
z[2, 10] = np.float32(3e38)
z[3] = (rng.normal(0, 1, size=V) * 1e30).astype(np.float32)
z[4] = np.float32(0.75); z[5, ::2] = np.float32(0.5)
raw = f32_to_bf16_bits(z) if dtype == "bf16" else z
params = [RowParams(temperature=1.0, top_p=0.9, seed=0, request_id=0), RowParams(temperature=1.0, top_p=0.3, seed=1, request_id=1),
          RowParams(temperature=1.0, top_p=0.9, seed=2, request_id=2), RowParams(temperature=1e30, top_k=300, seed=3, request_id=3),
          RowParams(temperature=1.0, top_k=2000, top_p=0.4, seed=4, request_id=4), RowParams(temperature=0.9, min_p=1.0, seed=5, request_id=5),
          RowParams(temperature=1e33, seed=6, request_id=6), RowParams(temperature=0.5, top_k=V - 1, min_p=0.2, seed=7, request_id=7)]
wl = Workload("edge", B, V, dtype, raw, [[]] * B, [[]] * B, params)
x = device_logits(wl)
orc = oracle_run(wl, 3)
full = make_sampler(wl).sample(x, 3)
for G in (1, 2, 3):
    outs, n, _ = sharded_inprocess(wl, x, G, step=3)
    o = outs[0]
    print("G", G, "rounds", n)
    for b in range(B):
        print("  row", b, "tok", int(o["tokens"][b]), "lp", float(o["logprobs"][b]), "flp", float(o["filtered_logprobs"][b]),
              "st", int(o["status"][b]), "| unsharded", int(full["tokens"][b]), float(full["logprobs"][b]),
              "| oracle", orc[b].token, orc[b].logprob, orc[b].filtered_logprob)
# merge only (no resolve rounds), G = 1 and 2
from paper_2506_22033_b200 import Sampler
from paper_2506_22033_b200.distributed import vocab_shard_bounds
for G in (1, 2):
    shs, recs = [], []
    for g in range(G):
        lo, hi = vocab_shard_bounds(V, G, g)
        sh = Sampler(V, B, max_history=64, dtype=dtype, vocab_offset=lo, vocab_local=hi - lo)
        sh.set_params(list(range(B)), params)
        rec = torch.empty(sh.record_bytes(B), dtype=torch.uint8, device="cuda")
        sh.sample_local(x[:, lo:hi], rec)
        shs.append(sh); recs.append(rec)
    torch.cuda.synchronize()
    r = recs[0].view(-1)[: shs[0].record_bytes(B) // B * 3].cpu().numpy()
    rb = shs[0].record_bytes(B) // B
    hdr = recs[0].view(-1)[2 * rb: 2 * rb + 48].cpu().numpy()
    print("row2 record hdr: m", hdr[0:4].view(np.float32), "flags", hdr[4:8].view(np.uint32), "s", hdr[8:16].view(np.float64), "R", hdr[16:24].view(np.float64), "n", hdr[24:28].view(np.uint32), "frontier", hex(int(hdr[32:40].view(np.uint64)[0])))
    o = shs[0].merge(torch.cat(recs), G, B, 3)
    torch.cuda.synchronize()
    print("merge G", G, "row2 tok", int(o["tokens"][2]), "lp", float(o["logprobs"][2]), "st", int(o["status"][2]))

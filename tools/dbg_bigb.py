"""Development: UNRESOLVED rows in the vocab-sharded paths at B > 2 x SMs (world 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import socket, torch, torch.distributed as dist
from tests._helpers import make_sampler
from workloads.synth import device_logits, make_workload
from paper_2506_22033_b200 import Sampler
from paper_2506_22033_b200.distributed import sample_vocab_sharded, sample_vocab_sharded_p2p, setup_peer_exchange
with socket.socket() as so:
    so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 320
wl = make_workload("c3", B=B, V=6000)
x = device_logits(wl)
for mode in ("nccl", "p2p", "local+merge"):
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    if mode == "p2p":
        setup_peer_exchange(s)
    bad = 0
    for step in range(20):
        if mode == "nccl":
            o = sample_vocab_sharded(s, x, step, resolve=False, append=True)
        elif mode == "p2p":
            o = sample_vocab_sharded_p2p(s, x, step, append=True)
        else:
            rec = torch.empty(s.record_bytes(B), dtype=torch.uint8, device="cuda")
            s.sample_local(x, rec)
            o = s.merge(rec, 1, B, step)
        torch.cuda.synchronize()
        st = o["status"].cpu()
        bad += int((st != 0).sum())
        if (st != 0).any() and bad < 5:
            print(mode, "step", step, "rows", (st != 0).nonzero().flatten().tolist()[:8], flush=True)
    print(mode, "B", B, "bad rows over 20 steps:", bad, flush=True)
dist.destroy_process_group()

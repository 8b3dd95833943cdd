"""The multi-GPU entry points on a real NCCL process group (world size 1: one GPU per gpurun call),
end to end against the float64 oracle, and captured in a CUDA graph.

* vocab-sharded (TP lm_head style): sample_local -> NCCL all_gather_into_tensor ->
  merge, on the whole vocabulary as the single shard;
* batch-row sharded: sample + the (token, logprob) all-gather.
The G = 2/4/8 split of the vocabulary is covered in test_gpu_parity.py with an in-process gather
(and the exchange plumbing at world size 2 with gloo in test_distributed.py).
"""
import os
import socket

import numpy as np
import pytest

from tests._helpers import assert_parity, make_sampler, oracle_run
from workloads.synth import device_logits, make_workload

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_vocab_sharded_nccl_world1_matches_oracle(nccl_group):
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import sample_vocab_sharded, vocab_shard_bounds
    wl = make_workload("c3", B=24, V=20000)
    lo, hi = vocab_shard_bounds(wl.V, 1, 0)
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    x = device_logits(wl)
    out = sample_vocab_sharded(s, x[:, lo:hi], 4)
    torch.cuda.synchronize()
    assert (out["status"] == 0).all()
    assert_parity(wl, out, oracle_run(wl, 4))


def test_vocab_sharded_step_in_cuda_graph(nccl_group):
    """The whole sharded step (local pass, NCCL all-gather, merge) captured once and replayed."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import sample_vocab_sharded
    wl = make_workload("c3", B=16, V=12000)
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    x = device_logits(wl)
    rb = s.record_bytes(wl.B)
    rec = torch.empty(rb, dtype=torch.uint8, device="cuda")
    gathered = torch.empty(rb, dtype=torch.uint8, device="cuda")
    out = s._outs(wl.B, None)
    eager = sample_vocab_sharded(s, x, 7, rec=rec, gathered=gathered, out=s._outs(wl.B, None))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        sample_vocab_sharded(s, x, 7, rec=rec, gathered=gathered, out=out)
    g.replay()
    torch.cuda.synchronize()
    for k in ("tokens", "logprobs", "status"):
        assert torch.equal(out[k], eager[k]), k
    assert_parity(wl, out, oracle_run(wl, 7))


def test_batch_row_sharded_nccl_world1_matches_oracle(nccl_group):
    import torch
    from paper_2506_22033_b200.distributed import batch_row_bounds, sample_batch_sharded
    wl = make_workload("c4", B=48, V=16000)
    lo, hi = batch_row_bounds(wl.B, 1, 0)
    s = make_sampler(wl)
    x = device_logits(wl)[lo:hi]
    o = sample_batch_sharded(s, x, 2, wl.B)
    torch.cuda.synchronize()
    assert torch.equal(o["tokens"], o["local"]["tokens"])
    assert_parity(wl, o["local"], oracle_run(wl, 2))
    assert np.isfinite(o["logprobs"].cpu().numpy()).all()


def test_vocab_sharded_unbounded_rows_nccl_and_graph(nccl_group):
    """NEXT-1 over NCCL: c2's top-p-only rows through sample_vocab_sharded (merge -> resolve rounds, each an
    all_gather_into_tensor), eager (adaptive round count) and captured in a CUDA graph with the fixed
    round count, both against the oracle."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import resolve_buffers, sample_vocab_sharded
    wl = make_workload("c2", B=8, V=30000)
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    x = device_logits(wl)
    eager = sample_vocab_sharded(s, x, 6)
    torch.cuda.synchronize()
    assert (eager["status"] == 0).all()
    assert_parity(wl, eager, oracle_run(wl, 6))
    rb = s.record_bytes(wl.B)
    rec = torch.empty(rb, dtype=torch.uint8, device="cuda")
    gathered = torch.empty(rb, dtype=torch.uint8, device="cuda")
    bufs = resolve_buffers(s, wl.B, 1, x.device)
    out = s._outs(wl.B, None)
    kw = dict(rec=rec, gathered=gathered, out=out, resolve_rounds=Sampler.resolve_max_rounds(), resolve_bufs=bufs)
    sample_vocab_sharded(s, x, 6, **kw)  # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        sample_vocab_sharded(s, x, 6, **kw)
    out["tokens"].fill_(-7)
    g.replay()
    torch.cuda.synchronize()
    for k in ("tokens", "logprobs", "status"):
        assert torch.equal(out[k], eager[k]), k


def test_peer_exchange_nccl_world1_graph_replays(nccl_group):
    """NEXT-2 on a real process group: setup_peer_exchange (handle all-gather) + sample_vocab_sharded_p2p,
    the step captured ONCE in a CUDA graph and replayed for several decode steps (per-row sequence numbers
    and record parities advance on the device): every replay equals the unsharded sampler's step."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import sample_vocab_sharded_p2p, setup_peer_exchange
    wl = make_workload("c3", B=16, V=12000)
    x = device_logits(wl)
    full = make_sampler(wl)
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    setup_peer_exchange(s)
    eager = sample_vocab_sharded_p2p(s, x, 0, append=True)
    ref = full.sample(x, 0, append=True)
    torch.cuda.synchronize()
    assert torch.equal(eager["tokens"], ref["tokens"])
    assert_parity(wl, eager, oracle_run(wl, 0))
    out = s._outs(wl.B, None)
    step = torch.tensor([5], dtype=torch.int64, device="cuda")
    s.set_step_source(step)  # the whole decode step in one graph: the Philox step advances per replay
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        sample_vocab_sharded_p2p(s, x, 0, out=out, append=True)
        step.add_(1)
    for i in range(3):
        g.replay()
        ref = full.sample(x, 5 + i, append=True)
        torch.cuda.synchronize()
        assert (out["status"] == 0).all()
        assert torch.equal(out["tokens"], ref["tokens"])


def _ipc_worker(rank, port, q):
    """One of two processes on the SAME GPU: CUDA IPC mapping of the other's exchange buffer (gloo for
    the handle exchange and the barriers).  Publish, barrier, merge: no kernel waits on the other process."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2506_22033_b200 import Sampler
        from paper_2506_22033_b200.distributed import setup_peer_exchange, vocab_shard_bounds
        wl = make_workload("c3", B=8, V=16000)
        x = device_logits(wl)
        lo, hi = vocab_shard_bounds(wl.V, 2, rank)
        s = Sampler(wl.V, wl.B, max_history=1024, dtype=wl.dtype, vocab_offset=lo, vocab_local=hi - lo)
        s.set_params(list(range(wl.B)), wl.params)
        for b in range(wl.B):
            s.set_history(b, wl.prompts[b], wl.outputs[b])
        setup_peer_exchange(s)
        ok = True
        for step in range(3):
            s.sample_exchange(x[:, lo:hi], step, phases=1)
            torch.cuda.synchronize()
            dist.barrier()
            o = s.sample_exchange(x[:, lo:hi], step, phases=2)
            torch.cuda.synchronize()
            dist.barrier()
            full = make_sampler(wl)
            ref = full.sample(x, step)
            torch.cuda.synchronize()
            ok = ok and bool((o["status"] == 0).all()) and torch.equal(o["tokens"], ref["tokens"])
        q.put((rank, ok))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_ipc_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def test_peer_exchange_with_resolve_rounds_in_one_graph(nccl_group):
    """The whole sharded decode step with unbounded rows through the peer exchange — candidate step, the
    fixed resolve round count, the step increment — captured once and replayed, == unsharded eager steps."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import sample_vocab_sharded_p2p, setup_peer_exchange
    wl = make_workload("c2", B=6, V=20000)
    x = device_logits(wl)
    full = make_sampler(wl, max_history=1024)
    s = Sampler(wl.V, wl.B, max_history=1024, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    setup_peer_exchange(s)
    eager = sample_vocab_sharded_p2p(s, x, 0, resolve=True)
    ref = full.sample(x, 0)
    torch.cuda.synchronize()
    assert (eager["status"] == 0).all() and torch.equal(eager["tokens"], ref["tokens"])
    step = torch.tensor([3], dtype=torch.int64, device="cuda")
    s.set_step_source(step)
    out = s._outs(wl.B, None)
    active = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        sample_vocab_sharded_p2p(s, x, 0, out=out, append=True, resolve=True,
                                 resolve_bufs=(None, None, active))
        step.add_(1)
    for i in range(3):
        g.replay()
        ref = full.sample(x, 3 + i, append=True)
        torch.cuda.synchronize()
        assert (out["status"] == 0).all()
        assert torch.equal(out["tokens"], ref["tokens"]), i


def test_peer_exchange_large_batch_uses_the_merge_kernel(nccl_group):
    """B > 2 x SMs: sampler_sample_exchange(phases=3) publishes, then merges in a separate kernel (no CTA
    waits for a row its GPU has not scheduled); decode steps with append == the unsharded sampler."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import sample_vocab_sharded_p2p, setup_peer_exchange
    wl = make_workload("c3", B=320, V=6000)
    x = device_logits(wl)
    full = make_sampler(wl, max_history=1024)
    s = Sampler(wl.V, wl.B, max_history=1024, max_top_k=40, dtype=wl.dtype, vocab_offset=0, vocab_local=wl.V)
    s.set_params(list(range(wl.B)), wl.params)
    for b in range(wl.B):
        s.set_history(b, wl.prompts[b], wl.outputs[b])
    setup_peer_exchange(s)
    for step in range(3):
        out = sample_vocab_sharded_p2p(s, x, step, append=True)
        ref = full.sample(x, step, append=True)
        torch.cuda.synchronize()
        assert s.last_launch_count() == 3
        st = out["status"].cpu()
        assert (st == 0).all(), (step, sorted(set(st.tolist())), (st != 0).nonzero().flatten().tolist()[:10])
        assert torch.equal(out["tokens"], ref["tokens"]), step

"""NEXT-1: vocab-sharded rows whose kept set is not bounded by the exchanged candidates (top-p-only,
min-p-only, unfiltered, top_k > max_top_k) finished by the resolve rounds (include/sampler.h,
csrc/resolve.cuh), against the float64 oracle.

G vocab slices run on one GPU in lock step with an in-process all-gather (torch.cat of the rank
payloads): every rank's round r is launched before the gather of round r, so no kernel ever waits on
another rank's kernel.  The NCCL path (world size 1) and its CUDA-graph capture are in
test_gpu_dist.py.
"""
import numpy as np
import pytest

from tests._helpers import assert_parity, oracle_run
from workloads.synth import RowParams, Workload, device_logits, make_workload, random_params

pytestmark = pytest.mark.gpu


def sharded_inprocess(wl, x, G, step, append=False, max_top_k=128, rounds=None, max_history=None):
    """Returns (per-rank outputs, exchanges, the per-rank samplers)."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import vocab_shard_bounds
    L = max_history or max(64, max(len(p) + len(o) for p, o in zip(wl.prompts, wl.outputs)) + 64)
    shards, xs, recs = [], [], []
    for r in range(G):
        lo, hi = vocab_shard_bounds(wl.V, G, r)
        sh = Sampler(wl.V, wl.B, max_history=L, max_top_k=max_top_k, dtype=wl.dtype, vocab_offset=lo,
                     vocab_local=hi - lo)
        sh.set_params(list(range(wl.B)), wl.params)
        for b in range(wl.B):
            if wl.prompts[b] or wl.outputs[b]:
                sh.set_history(b, wl.prompts[b], wl.outputs[b])
        xs.append(x[:, lo:hi])
        rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
        sh.sample_local(xs[-1], rec)
        recs.append(rec)
        shards.append(sh)
    gathered = torch.cat(recs)
    outs = [sh.merge(gathered, G, wl.B, step, append=append) for sh in shards]
    pays = [torch.empty(sh.resolve_bytes(wl.B), dtype=torch.uint8, device="cuda") for sh in shards]
    act = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in shards]
    for g, sh in enumerate(shards):
        sh.resolve_round(xs[g], step, 0, None, G, g, pays[g], outs[g], append=append, active=act[g])
    n = 0
    while (rounds is None and int(act[0].item()) > 0) or (rounds is not None and n < rounds):
        gathered = torch.cat(pays)
        n += 1
        for g, sh in enumerate(shards):
            sh.resolve_round(xs[g], step, n, gathered, G, g, pays[g], outs[g], append=append, active=act[g])
    torch.cuda.synchronize()
    assert all(int(a.item()) == 0 for a in act)
    return outs, n, shards


def _check_all_ranks(wl, outs, orc):
    import torch
    for o in outs[1:]:  # every rank computed the same outputs
        for k in ("tokens", "logprobs", "filtered_logprobs", "status"):
            assert torch.equal(o[k], outs[0][k]), k
    assert_parity(wl, outs[0], orc)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_c2_top_p_only_rows_resolved(G):
    wl = make_workload("c2", B=12, V=40000)
    x = device_logits(wl)
    outs, n, _ = sharded_inprocess(wl, x, G, step=3)
    assert (outs[0]["status"] == 0).all()
    assert 3 <= n <= 20, n
    _check_all_ranks(wl, outs, oracle_run(wl, 3))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_mixed_unbounded_params(dtype):
    """Every kind of row in one batch: top-p only, min-p only, unfiltered, top_k > max_top_k (alone and
    with top-p / min-p), and rows the merge decides itself (greedy, top-k 40)."""
    rng = np.random.default_rng(7)
    wl = make_workload("c2", B=16, V=24000, dtype=dtype)
    P = [RowParams(temperature=1.0, top_p=0.9), RowParams(temperature=0.8, min_p=0.02),
         RowParams(temperature=1.2), RowParams(temperature=0.7, top_k=300),
         RowParams(temperature=1.0, top_k=1000, top_p=0.8), RowParams(temperature=0.9, top_k=500, min_p=0.1),
         RowParams(temperature=0.0), RowParams(temperature=0.7, top_k=40, top_p=0.9),
         RowParams(temperature=1.0, top_p=0.5, min_p=0.05), RowParams(temperature=0.3, top_p=0.99),
         RowParams(temperature=2.0, top_k=129), RowParams(temperature=1.0, top_p=0.999)]
    for b in range(wl.B):
        p = P[b] if b < len(P) else random_params(rng, b, wl.V)
        p.seed, p.request_id = 100 + b, 7000 + b
        if b % 2:
            p.repetition_penalty, p.presence_penalty, p.frequency_penalty = 1.2, 0.3, 0.1
        wl.params[b] = p
    x = device_logits(wl)
    for G in (1, 3, 8):
        outs, n, _ = sharded_inprocess(wl, x, G, step=5)
        assert (outs[0]["status"] == 0).all(), outs[0]["status"]
        _check_all_ranks(wl, outs, oracle_run(wl, 5))


def test_ties_and_flat_rows_deep_rounds():
    """All-equal rows (one value: the search descends into the id bits), a few distinct values, an
    increasing ramp, -inf-masked rows with fewer than top_k finite logits."""
    B, V = 8, 20000
    z = np.zeros((B, V), dtype=np.float32)
    z[0] = 1.5
    z[1, ::3] = 2.0
    z[2] = np.arange(V, dtype=np.float32) * np.float32(1e-4)
    z[3] = -np.inf
    z[3, 100:160] = np.linspace(-1, 1, 60, dtype=np.float32)
    z[4] = (np.arange(V) % 5).astype(np.float32)
    z[5] = -np.inf
    z[5, 7] = 0.0
    z[6] = np.float32(-3.0)
    z[6, 19999] = 0.0
    z[7] = np.arange(V, dtype=np.float32)[::-1] * np.float32(-1e-3)
    params = [RowParams(temperature=1.0, top_p=0.5, seed=b, request_id=b) for b in range(B)]
    params[1] = RowParams(temperature=1.0, top_k=5000, seed=1, request_id=1)
    params[3] = RowParams(temperature=1.0, top_k=200, seed=3, request_id=3)
    params[4] = RowParams(temperature=0.5, top_k=9000, top_p=0.7, seed=4, request_id=4)
    params[5] = RowParams(temperature=1.0, min_p=0.5, seed=5, request_id=5)
    params[6] = RowParams(temperature=1.0, seed=6, request_id=6)
    params[7] = RowParams(temperature=0.01, top_p=0.95, seed=7, request_id=7)
    wl = Workload("ties", B, V, "f32", z, [[]] * B, [[]] * B, params)
    x = device_logits(wl)
    for G in (1, 2, 5):
        outs, n, _ = sharded_inprocess(wl, x, G, step=2)
        assert (outs[0]["status"] == 0).all(), outs[0]["status"]
        _check_all_ranks(wl, outs, oracle_run(wl, 2))


def test_resolve_fixed_rounds_and_append():
    """The fixed round count (graph-capturable) gives the same outputs as the adaptive loop; with
    append the resolved tokens enter every rank's history (replicated tables)."""
    import torch
    wl = make_workload("c2", B=6, V=16000)
    x = device_logits(wl)
    from paper_2506_22033_b200 import Sampler
    ad, n, _ = sharded_inprocess(wl, x, 2, step=1)
    fx, n2, shards = sharded_inprocess(wl, x, 2, step=1, rounds=Sampler.resolve_max_rounds(), append=True)
    assert n2 == Sampler.resolve_max_rounds() and n <= n2
    for k in ("tokens", "logprobs", "status"):
        assert torch.equal(ad[0][k], fx[0][k]), k
    toks = fx[0]["tokens"].cpu().tolist()
    for sh in shards:
        for b in range(wl.B):
            assert sh.get_history(b)["output"] == list(wl.outputs[b]) + [toks[b]]


def test_full_size_c2_vocab_sharded_sampled_rows():
    """BASELINE's c2 size (B=64, V=152064) vocab-sharded over 8 slices; sampled rows vs the oracle."""
    wl = make_workload("c2")
    x = device_logits(wl)
    outs, n, _ = sharded_inprocess(wl, x, 8, step=11)
    assert (outs[0]["status"] == 0).all()
    rows = list(range(0, 64, 7))
    _check_all_ranks(wl, [outs[0]], oracle_run(wl, 11, rows=rows))


# ---------------------------------------------------------------- NEXT-2: one-shot peer exchange
def _exchange_shards(wl, G, timeout_ms=0, max_top_k=128):
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import vocab_shard_bounds
    L = max(64, max(len(p) + len(o) for p, o in zip(wl.prompts, wl.outputs)) + 64)
    shards, bounds = [], []
    for g in range(G):
        lo, hi = vocab_shard_bounds(wl.V, G, g)
        sh = Sampler(wl.V, wl.B, max_history=L, max_top_k=max_top_k, dtype=wl.dtype, vocab_offset=lo,
                     vocab_local=hi - lo)
        sh.set_params(list(range(wl.B)), wl.params)
        for b in range(wl.B):
            if wl.prompts[b] or wl.outputs[b]:
                sh.set_history(b, wl.prompts[b], wl.outputs[b])
        shards.append(sh)
        bounds.append((lo, hi))
    bases = [sh.exchange_init(G, g, timeout_ms)[1] for g, sh in enumerate(shards)]
    for sh in shards:
        sh.exchange_set_peers(bases)
    return shards, bounds


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_peer_exchange_inprocess_decode_steps(G):
    """G ranks of one process on one GPU in lock step (every rank's publish before any rank's merge):
    records stored into every rank's buffer by phase 1, flags, double-buffered parities over several
    decode steps with append — tokens equal the unsharded sampler's at every step, step 0 vs the oracle."""
    import torch
    from tests._helpers import make_sampler
    wl = make_workload("c3", B=24, V=30000)
    x = device_logits(wl)
    full = make_sampler(wl)
    shards, bounds = _exchange_shards(wl, G)
    for step in range(4):
        ref = full.sample(x, step, append=True)
        for g, sh in enumerate(shards):
            sh.sample_exchange(x[:, bounds[g][0]:bounds[g][1]], step, append=True, phases=1)
        outs = [sh.sample_exchange(x[:, bounds[g][0]:bounds[g][1]], step, append=True, phases=2)
                for g, sh in enumerate(shards)]
        torch.cuda.synchronize()
        for o in outs:
            assert (o["status"] == 0).all()
            assert torch.equal(o["tokens"], ref["tokens"])
            assert torch.allclose(o["logprobs"], ref["logprobs"], rtol=1e-5, atol=1e-6)
        if step == 0:
            assert_parity(wl, outs[0], oracle_run(wl, 0))
    for sh in shards:  # replicated histories stayed in step with the unsharded handle
        for b in (0, wl.B - 1):
            assert sh.get_history(b)["output"] == full.get_history(b)["output"]


def test_peer_exchange_timeout_reports_rows():
    """A merge whose peer never publishes reports SAMPLER_ROW_EXCHANGE_TIMEOUT after the timeout instead of
    hanging the GPU."""
    import torch
    from paper_2506_22033_b200 import ROW_EXCHANGE_TIMEOUT
    wl = make_workload("c3", B=4, V=8000)
    x = device_logits(wl)
    shards, bounds = _exchange_shards(wl, 2, timeout_ms=50)
    shards[0].sample_exchange(x[:, bounds[0][0]:bounds[0][1]], 0, phases=1)   # rank 1 never publishes
    o = shards[0].sample_exchange(x[:, bounds[0][0]:bounds[0][1]], 0, phases=2)
    torch.cuda.synchronize()
    assert (o["status"] == ROW_EXCHANGE_TIMEOUT).all() and (o["tokens"] == -1).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_sharded_edge_rows(dtype):
    """The vocab-sharded path (merge + resolve rounds) on the edge rows of the unsharded suite: subnormal /
    signed-zero logits, values near the binary32 limit, huge temperatures, all-equal rows, min_p = 1."""
    B, V = 8, 9000
    rng = np.random.default_rng(17)
    z = rng.normal(0, 2, size=(B, V)).astype(np.float32)
    z[0] = (rng.integers(-50, 50, size=V) * np.float32(1e-41)).astype(np.float32)
    z[1] = np.float32(0.0)
    z[1, ::2] = np.float32(-0.0)
    z[2, 10] = np.float32(3e38)
    z[3] = (rng.normal(0, 1, size=V) * 1e30).astype(np.float32)
    z[4] = np.float32(0.75)
    z[5, ::2] = np.float32(0.5)
    if dtype == "bf16":
        from workloads.synth import f32_to_bf16_bits
        raw = f32_to_bf16_bits(z)
    else:
        raw = z
    params = [RowParams(temperature=1.0, top_p=0.9, seed=0, request_id=0),
              RowParams(temperature=1.0, top_p=0.3, seed=1, request_id=1),
              RowParams(temperature=1.0, top_p=0.9, seed=2, request_id=2),
              RowParams(temperature=1e30, top_k=300, seed=3, request_id=3),
              RowParams(temperature=1.0, top_k=2000, top_p=0.4, seed=4, request_id=4),
              RowParams(temperature=0.9, min_p=1.0, seed=5, request_id=5),
              RowParams(temperature=1e33, seed=6, request_id=6),
              RowParams(temperature=0.5, top_k=V - 1, min_p=0.2, seed=7, request_id=7)]
    wl = Workload("edge", B, V, dtype, raw, [[]] * B, [[]] * B, params)
    x = device_logits(wl)
    for G in (2, 3):
        outs, n, _ = sharded_inprocess(wl, x, G, step=3)
        assert (outs[0]["status"] == 0).all(), outs[0]["status"]
        _check_all_ranks(wl, outs, oracle_run(wl, 3))


@pytest.mark.parametrize("G", [1, 2, 4])
def test_peer_exchange_resolve_rounds(G):
    """NEXT-1 + NEXT-2: unbounded rows (c2 top-p-only, mixed) resolved with every payload through the peer
    exchange (sampler_resolve_round_exchange: flags, parities, no collective), G ranks of one process in lock
    step over two decode steps with append, vs the oracle replaying the grown histories."""
    import torch
    wl = make_workload("c2", B=6, V=24000)
    wl.params[1] = RowParams(temperature=0.8, min_p=0.02, seed=3, request_id=3)
    wl.params[2] = RowParams(temperature=0.7, top_k=700, top_p=0.9, seed=4, request_id=4)
    wl.params[3] = RowParams(temperature=0.0, seed=5, request_id=5)
    x = device_logits(wl)
    shards, bounds = _exchange_shards(wl, G)
    xs = [x[:, lo:hi] for lo, hi in bounds]
    outputs = [list(o) for o in wl.outputs]
    for step in range(2):
        for g, sh in enumerate(shards):
            sh.sample_exchange(xs[g], step, append=True, phases=1)
        outs = [sh.sample_exchange(xs[g], step, append=True, phases=2) for g, sh in enumerate(shards)]
        act = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in shards]
        r = 0
        while True:
            for g, sh in enumerate(shards):
                sh.resolve_round_exchange(xs[g], step, r, outs[g], append=True, active=act[g])
            torch.cuda.synchronize()
            if int(act[0].item()) == 0:
                break
            r += 1
            assert r <= 20
        cur = Workload(wl.name, wl.B, wl.V, wl.dtype, wl.raw, wl.prompts, [list(o) for o in outputs], wl.params)
        assert (outs[0]["status"] == 0).all(), outs[0]["status"]
        _check_all_ranks(cur, outs, oracle_run(cur, step))
        for b, t in enumerate(outs[0]["tokens"].cpu().tolist()):
            outputs[b].append(int(t))
    for sh in shards:
        for b in range(wl.B):
            assert sh.get_history(b)["output"] == outputs[b]

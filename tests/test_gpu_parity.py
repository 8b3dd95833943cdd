"""CUDA path vs the float64 oracle, element by element, through the C ABI.

Sizes: small enough for the oracle to finish in seconds yet spanning many 2 KB tiles, many warp
spans per row, ragged row tails (ld > V) and the degenerate cases; plus BASELINE.json's full
sizes on sampled rows.
"""
import math

import numpy as np
import pytest

from tests._helpers import assert_parity, device_logits, make_sampler, oracle_run, oracle_params
from workloads.synth import RowParams, Workload, make_workload, random_params, gen_logits

pytestmark = pytest.mark.gpu


def _run(wl, step=0, ld=None, q=False, **kw):
    s = make_sampler(wl, **kw)
    x = device_logits(wl, ld=ld)
    if q:
        out = s.debug_distribution(x, step)
        out["status"] = None
        out["filtered_logprobs"] = None
    else:
        out = s.sample(x, step)
    import torch
    torch.cuda.synchronize()
    return s, out


def test_c1_full_config_with_distribution():
    wl = make_workload("c1")
    orc = oracle_run(wl, step=0, want_q=True)
    s, out = _run(wl, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s2, out2 = _run(wl)
    assert_parity(wl, out2, oracle_run(wl, 0))


@pytest.mark.parametrize("cfg", ["c3", "c5", "c2", "c4"])
def test_small_batch_full_vocab(cfg):
    wl = make_workload(cfg, B=12)
    orc = oracle_run(wl, step=3)
    s, out = _run(wl, step=3)
    assert_parity(wl, out, orc)


@pytest.mark.parametrize("V,ld,dtype", [(1, 8, "bf16"), (7, 16, "f32"), (100, 104, "bf16"), (1001, 1008, "bf16"),
                                        (5003, 5008, "f32"), (32000, 32000, "bf16"), (40000, 40008, "f32")])
def test_random_params_ragged_shapes(V, ld, dtype):
    rng = np.random.default_rng(V)
    B = 24
    raw = gen_logits(rng, B, V, dtype)
    prompts, outputs = [], []
    for b in range(B):
        n = int(rng.integers(0, 40))
        toks = rng.integers(0, V, size=n).tolist()
        prompts.append(toks[: n // 2])
        outputs.append(toks[n // 2:])
    params = [random_params(rng, b, V) for b in range(B)]
    wl = Workload("rand", B, V, dtype, raw, prompts, outputs, params)
    orc = oracle_run(wl, step=11, want_q=True)
    s, out = _run(wl, step=11, ld=ld, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s, out = _run(wl, step=11, ld=ld)
    assert_parity(wl, out, oracle_run(wl, 11))


@pytest.mark.parametrize("cfg", ["c3", "c2", "c1"])
def test_linear_penalty_mode(cfg):
    """The paper-literal subtractive penalty (R1 LINEAR)."""
    wl = make_workload(cfg, B=min(16, make_workload(cfg).B))
    s, out = _run(wl, step=3, mode=1)
    assert_parity(wl, out, oracle_run(wl, 3, mode=1))


def test_greedy_and_topk1_bit_exact_with_ties():
    rng = np.random.default_rng(5)
    B, V = 64, 20000
    z = rng.integers(-20, 20, size=(B, V)).astype(np.float32)  # massive exact ties
    params = []
    for b in range(B):
        if b % 2:
            params.append(RowParams(temperature=0.0, seed=b, request_id=b))
        else:
            params.append(RowParams(temperature=0.9, top_k=1, seed=b, request_id=b))
    wl = Workload("ties", B, V, "f32", z, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=0)
    s, out = _run(wl)
    assert_parity(wl, out, orc)
    zp = z  # no penalties
    assert np.array_equal(out["tokens"].cpu().numpy(), np.argmax(zp, axis=1))


def test_row_faults_nan_inf_all_neg_inf():
    rng = np.random.default_rng(6)
    B, V = 6, 3000
    z = rng.normal(size=(B, V)).astype(np.float32)
    z[0, 17] = np.nan
    z[1, 2999] = np.inf
    z[2, :] = -np.inf
    z[3, :-1] = -np.inf  # only the last id is finite
    z[4, ::2] = -np.inf
    params = [RowParams(temperature=1.0, top_k=10, seed=b) for b in range(B)]
    params[5] = RowParams(temperature=1.0, top_p=0.5, seed=5)
    wl = Workload("faults", B, V, "f32", z, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=0)
    s, out = _run(wl)
    assert_parity(wl, out, orc)
    assert out["tokens"][3].item() == V - 1
    assert math.isnan(out["logprobs"][0].item())


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_topk_only_rows_with_fewer_than_k_finite_logits(dtype):
    """with every row top-k-only the exact multi-pass kernel is not launched; rows with
    fewer finite logits than k (constrained decoding masks) must still be decided, with
    K1 = every finite id; also a row whose finite logits lie far below one huge logit."""
    from workloads.synth import f32_to_bf16_bits
    rng = np.random.default_rng(78)
    B, V = 8, 4000
    z = rng.normal(size=(B, V)).astype(np.float32)
    z[1, :] = -np.inf
    z[1, [5, 77, 1234]] = [0.5, 1.5, -2.0]            # 3 finite logits, k = 40
    z[2, :-39] = -np.inf                               # 39 finite logits, k = 40
    z[3, :] = -np.inf
    z[3, 100] = 3.0                                    # a single finite logit
    z[4, 7] = 3.0e4                                    # one huge logit, the rest far below it
    z[5, ::3] = -np.inf
    raw = f32_to_bf16_bits(z) if dtype == "bf16" else z
    params = [RowParams(temperature=0.9, top_k=40, top_p=0.95 if b % 2 else 1.0, seed=b, request_id=b)
              for b in range(B)]
    wl = Workload("fewfinite", B, V, dtype, raw, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=2)
    s, out = _run(wl, step=2)
    assert s.last_launch_count() == 2  # stream + select only: nothing may stay pending
    assert_parity(wl, out, orc)
    assert out["tokens"][3].item() == 100


def test_determinism_bit_identical():
    import torch
    wl = make_workload("c4", B=64)
    s = make_sampler(wl)
    x = device_logits(wl)
    a = s.sample(x, 5)
    a = {k: v.clone() for k, v in a.items()}
    b = s.sample(x, 5)
    torch.cuda.synchronize()
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_cuda_graph_replay_equals_eager_and_oracle():
    """bench.py replays the step from CUDA graphs: a captured step (programmatic dependent launch
    inside the graph, in-kernel history append) must give the eager call's bits, and the oracle's
    tokens on the grown histories."""
    import torch
    wl = make_workload("c3", B=64)
    x = device_logits(wl)
    se = make_sampler(wl, max_history=1024)
    sg = make_sampler(wl, max_history=1024)
    oute = [{k: v.clone() for k, v in se.sample(x, i, append=True).items()} for i in range(3)]
    outg = sg._outs(wl.B, None)
    res = []  # (the step id is baked into a graph: one graph per step)
    for i in range(3):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.Stream()):
            sg.sample(x, i, append=True, out=outg)
        g.replay()
        torch.cuda.synchronize()
        res.append({k: v.clone() for k, v in outg.items()})
    for i in range(3):
        for k in ("tokens", "logprobs", "filtered_logprobs", "status"):
            assert torch.equal(oute[i][k], res[i][k]), (i, k)
    # histories grew identically
    for b in (0, 17, 63):
        assert se.get_history(b) == sg.get_history(b)


def test_history_append_matches_sequential_oracle():
    """Decode 6 steps with in-kernel history append; the oracle replays with the grown history."""
    import torch
    wl = make_workload("c3", B=8, V=20000)
    s = make_sampler(wl, max_history=1024)
    x = device_logits(wl)
    outputs = [list(o) for o in wl.outputs]
    for step in range(6):
        out = s.sample(x, step, append=True)
        torch.cuda.synchronize()
        cur = Workload(wl.name, wl.B, wl.V, wl.dtype, wl.raw, wl.prompts, [list(o) for o in outputs], wl.params)
        orc = oracle_run(cur, step)
        assert_parity(cur, out, orc)
        toks = out["tokens"].cpu().numpy()
        for b in range(wl.B):
            if orc[b].token == toks[b]:
                outputs[b].append(int(toks[b]))
            else:  # flagged mismatch: follow the GPU so histories stay aligned
                outputs[b].append(int(toks[b]))
    for b in range(wl.B):
        h = s.get_history(b)
        assert h["output"] == outputs[b]
        # incremental unique table == recount (SPEC S:248 buffer consistency)
        ids = sorted(set(wl.prompts[b]) | set(outputs[b]))
        assert h["uniq_ids"] == ids
        assert h["uniq_counts"] == [outputs[b].count(i) for i in ids]
        assert h["uniq_in_prompt"] == [int(i in set(wl.prompts[b])) for i in ids]


def test_slots_and_device_params_and_seeds():
    import torch
    from paper_2506_22033_b200 import params_to_device
    wl = make_workload("c4", B=16)
    s = make_sampler(wl, max_batch=40)
    # map row b -> slot 39-b, with histories moved accordingly
    for b in range(wl.B):
        s.set_history(39 - b, wl.prompts[b], wl.outputs[b])
    slots = torch.tensor([39 - b for b in range(wl.B)], dtype=torch.int32, device="cuda")
    pd = params_to_device(wl.params)
    seeds = torch.tensor([p.seed + 1000 for p in wl.params], dtype=torch.int64, device="cuda")
    x = device_logits(wl)
    out = s.sample(x, 2, slots=slots, params=pd, seeds=seeds)
    torch.cuda.synchronize()
    wl2 = Workload(wl.name, wl.B, wl.V, wl.dtype, wl.raw, wl.prompts, wl.outputs,
                   [RowParams(**{**p.__dict__, "seed": p.seed + 1000}) for p in wl.params])
    assert_parity(wl2, out, oracle_run(wl2, 2))


def test_invalid_device_slots_and_params_give_row_status():
    """Device-supplied slots / params are not seen by the host: an out-of-range slot or a parameter
    set that sampler_set_params rejects gives SAMPLER_ROW_INVALID for that row (token -1, NaN
    logprob, no append), every other row is unaffected (ADVICE / VERDICT r1 item 11)."""
    import torch
    from paper_2506_22033_b200 import ROW_INVALID, params_to_device
    wl = make_workload("c3", B=10, V=9000)
    s = make_sampler(wl, max_batch=16)
    x = device_logits(wl)
    params = [RowParams(**p.__dict__) for p in wl.params]
    params[2].temperature = -1.0
    params[3].top_p = 0.0
    params[4].repetition_penalty = 0.0   # OPENAI_CTRL needs > 0
    params[5].min_p = float("nan")
    slots = torch.arange(wl.B, dtype=torch.int32, device="cuda")
    slots[6] = 16                          # == max_batch: out of range
    slots[7] = -3
    before = [s.get_history(b) for b in range(wl.B)]
    out = s.sample(x, 1, slots=slots, params=params_to_device(params), append=True)
    torch.cuda.synchronize()
    st = out["status"].cpu().tolist()
    tok = out["tokens"].cpu().tolist()
    bad = {2, 3, 4, 5, 6, 7}
    for b in range(wl.B):
        if b in bad:
            assert st[b] == ROW_INVALID and tok[b] == -1, (b, st[b], tok[b])
            assert math.isnan(out["logprobs"][b].item())
        else:
            assert st[b] == 0
    for b in (2, 3, 4, 5):                 # invalid rows appended nothing to their (valid) slots
        assert s.get_history(b) == before[b]
    orc = oracle_run(wl, 1, rows=[b for b in range(wl.B) if b not in bad])
    assert_parity(wl, out, orc)


def test_vocab_sharded_equals_unsharded_fake_allgather():
    """G vocab slices on one GPU with an in-process all-gather (torch.cat) == unsharded sampling."""
    import torch
    from paper_2506_22033_b200 import Sampler
    from paper_2506_22033_b200.distributed import vocab_shard_bounds
    wl = make_workload("c3", B=32, V=30000)
    x = device_logits(wl)
    full = make_sampler(wl)
    ref = full.sample(x, 9)
    torch.cuda.synchronize()
    for G in (2, 4, 8):
        shards = []
        recs = []
        for r in range(G):
            lo, hi = vocab_shard_bounds(wl.V, G, r)
            sh = Sampler(wl.V, wl.B, max_history=1024, max_top_k=128, dtype=wl.dtype, vocab_offset=lo,
                         vocab_local=hi - lo)
            sh.set_params(list(range(wl.B)), wl.params)
            for b in range(wl.B):
                sh.set_history(b, wl.prompts[b], wl.outputs[b])
            rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
            sh.sample_local(x[:, lo:hi], rec)
            shards.append(sh)
            recs.append(rec)
        gathered = torch.cat(recs)
        outs = [sh.merge(gathered, G, wl.B, 9) for sh in shards]
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o["tokens"], ref["tokens"])
            assert torch.allclose(o["logprobs"], ref["logprobs"], rtol=1e-5, atol=1e-6)
            assert (o["status"] == 0).all()


def test_vocab_sharded_top_p_only_rows_report_unresolved():
    import torch
    from paper_2506_22033_b200 import Sampler, ROW_UNRESOLVED
    wl = make_workload("c2", B=4, V=16000)
    x = device_logits(wl)
    recs, shs = [], []
    for r in range(2):
        sh = Sampler(wl.V, wl.B, max_history=1024, dtype=wl.dtype, vocab_offset=r * 8000, vocab_local=8000)
        sh.set_params(list(range(wl.B)), wl.params)
        rec = torch.empty(sh.record_bytes(wl.B), dtype=torch.uint8, device="cuda")
        sh.sample_local(x[:, r * 8000:(r + 1) * 8000], rec)
        recs.append(rec)
        shs.append(sh)
    o = shs[0].merge(torch.cat(recs), 2, wl.B, 0)
    torch.cuda.synchronize()
    st = o["status"].cpu().numpy()
    assert set(st.tolist()) <= {0, ROW_UNRESOLVED}


def test_full_size_c3_sampled_rows():
    """BASELINE configs[2] at full size (B=256, V=152064) in the bench launch configuration;
    the oracle checks a sample of rows one by one."""
    wl = make_workload("c3")
    s, out = _run(wl, step=1)
    rows = list(range(0, 256, 16)) + [255]
    orc = oracle_run(wl, 1, rows=rows)
    assert_parity(wl, out, orc)
    st = out["status"].cpu().numpy()
    assert (st == 0).all()
    assert s.last_launch_count() == 2  # stream + row merge; the exact multi-pass kernel is not needed


def test_full_size_c2_sampled_rows():
    wl = make_workload("c2")
    s, out = _run(wl, step=1)
    orc = oracle_run(wl, 1, rows=list(range(0, 64, 8)))
    assert_parity(wl, out, orc)


def test_full_size_c4_sampled_rows():
    wl = make_workload("c4")
    s, out = _run(wl, step=1)
    orc = oracle_run(wl, 1, rows=list(range(0, 1024, 97)))
    assert_parity(wl, out, orc)


def test_c5_latency_batches():
    for B in (1, 2, 4, 8, 16, 32):
        wl = make_workload("c5", B=B)
        s, out = _run(wl, step=4)
        assert_parity(wl, out, oracle_run(wl, 4))


def test_adversarial_floods_all_equal_and_increasing():
    """Candidate floods: all-equal rows (every element ties with the threshold) and strictly
    increasing rows (every element beats the running threshold) — the overflow/shrink paths."""
    B, V = 8, 40000
    z = np.zeros((B, V), dtype=np.float32)
    z[2] = np.arange(V, dtype=np.float32) * np.float32(1e-3)          # increasing
    z[3] = -np.arange(V, dtype=np.float32) * np.float32(1e-3)         # decreasing
    z[4] = np.float32(1.5)
    z[5, ::7] = np.float32(2.0)
    z[6] = np.arange(V, dtype=np.float32) * np.float32(1e-3)
    z[7] = np.float32(-1.0)
    params = [RowParams(temperature=0.7, top_k=40, seed=b, request_id=b) for b in range(B)]
    params[1] = RowParams(temperature=1.0, top_k=128, top_p=0.5, seed=1)
    params[6] = RowParams(temperature=0.0, seed=6)
    params[7] = RowParams(temperature=1.0, top_k=100, min_p=0.5, seed=7)
    wl = Workload("flood", B, V, "f32", z, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=2, want_q=True)
    s, out = _run(wl, step=2, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s, out = _run(wl, step=2)
    assert_parity(wl, out, oracle_run(wl, 2))


@pytest.mark.parametrize("n_hist", [700, 1800, 5000])
def test_long_histories_penalties(n_hist):
    """Unique-token tables beyond the speculative RT1 load (1024 entries), beyond the smem staging
    (2048: the selection reads the table from global), with all three penalties and top-k / top-p /
    min-p rows."""
    rng = np.random.default_rng(11 + n_hist)
    B, V = 8, 20000
    z = gen_logits(rng, B, V, "bf16")
    prompts, outputs = [], []
    for b in range(B):
        h = rng.choice(V, size=n_hist, replace=b % 2 == 0).tolist()
        prompts.append(h[: n_hist // 2])
        outputs.append(h[n_hist // 2:])
    params = []
    for b in range(B):
        params.append(RowParams(temperature=0.8, top_k=[0, 40, 128, 5][b % 4], top_p=[0.9, 1.0, 0.95, 1.0][b % 4],
                                min_p=[0.0, 0.0, 0.02, 0.1][b % 4], repetition_penalty=1.3, presence_penalty=0.4,
                                frequency_penalty=0.2, seed=100 + b, request_id=b))
    wl = Workload("longhist", B, V, "bf16", z, prompts, outputs, params)
    orc = oracle_run(wl, step=3)
    s, out = _run(wl, step=3)
    assert_parity(wl, out, orc)


@pytest.mark.parametrize("n_hist", [32768, 131072])
def test_very_long_histories_full_vocab(n_hist):
    """NEXT-4 (L_max <= 128K): 32K / 128K-token histories at the c3 vocabulary, every
    penalty, top-k / top-p / min-p / unfiltered rows, three steps with in-kernel appends against the
    oracle's recount."""
    import torch
    rng = np.random.default_rng(n_hist)
    B, V = 4, 152064
    z = gen_logits(rng, B, V, "bf16")
    prompts, outputs = [], []
    for b in range(B):
        # a Zipf-like stream over the vocabulary (repeats) plus a pool of likely tokens
        h = np.concatenate([rng.zipf(1.1, size=n_hist // 2) % V, rng.integers(0, V, size=n_hist - n_hist // 2)])
        rng.shuffle(h)
        h = h.astype(np.int64).tolist()
        prompts.append(h[: n_hist - 64])
        outputs.append(h[n_hist - 64:])
    params = [RowParams(temperature=0.8, top_k=40, top_p=0.9, min_p=0.05, repetition_penalty=1.2,
                        presence_penalty=0.4, frequency_penalty=0.1, seed=1, request_id=0),
              RowParams(temperature=1.0, top_p=0.95, repetition_penalty=1.1, presence_penalty=0.3,
                        frequency_penalty=0.2, seed=2, request_id=1),
              RowParams(temperature=0.7, min_p=0.1, repetition_penalty=1.3, seed=3, request_id=2),
              RowParams(temperature=1.0, frequency_penalty=0.05, seed=4, request_id=3)]
    wl = Workload("hist", B, V, "bf16", z, prompts, outputs, params)
    s = make_sampler(wl, max_history=n_hist + 16)
    x = device_logits(wl)
    for step in range(3):
        out = s.sample(x, step, append=True)
        torch.cuda.synchronize()
        assert_parity(wl, out, oracle_run(wl, step))
        tok = out["tokens"].cpu().numpy()
        for b in range(B):  # the oracle's history follows the sampled tokens
            wl.outputs[b] = wl.outputs[b] + [int(tok[b])]
    for b in range(B):
        h = s.get_history(b)
        assert h["output"] == wl.outputs[b]
        ids = sorted(set(wl.prompts[b]) | set(wl.outputs[b]))
        assert h["uniq_ids"] == ids



@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_temperature_edges_and_subnormal_logits(dtype):
    """tau at the greedy boundary (binary32 9.99e-6 < 1e-5 <= 1e-5: R5), very small tau (a rebase of the lane
    reference at almost every group, weights underflowing to 0 past the max), very large tau, and rows of
    subnormal / signed-zero logits; tokens, logprobs and the whole filtered distribution q vs the oracle."""
    B, V = 12, 5000
    rng = np.random.default_rng(99)
    z = rng.normal(0, 2, size=(B, V)).astype(np.float32)
    z[6] = (rng.integers(-50, 50, size=V) * np.float32(1e-41)).astype(np.float32)   # subnormals
    z[7] = np.float32(0.0)
    z[7, ::2] = np.float32(-0.0)
    z[7, 17] = np.float32(1e-45)                                                  # smallest subnormal wins
    z[8] = np.where(rng.random(V) < 0.5, np.float32(-1e-44), np.float32(3e-39))
    z[9] = np.float32(-np.inf)
    z[9, 4000:4003] = np.float32([1e-40, -2e-40, 5e-41])
    if dtype == "bf16":
        from workloads.synth import f32_to_bf16_bits
        raw = f32_to_bf16_bits(z)
    else:
        raw = z
    taus = [9.99e-6, 1e-5, 1.0001e-5, 1e-4, 0.01, 100.0, 1.0, 1.0, 0.5, 1.0, 2e-5, 50.0]
    params = [RowParams(temperature=t, top_p=0.9 if b % 3 == 0 else 1.0, top_k=20 if b % 3 == 1 else 0,
                        seed=b, request_id=b) for b, t in enumerate(taus)]
    wl = Workload("tau", B, V, dtype, raw, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=4, want_q=True)
    s, out = _run(wl, step=4, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s, out = _run(wl, step=4)
    assert_parity(wl, out, oracle_run(wl, 4))


def test_q_full_vocab_for_exact_kernel_rows():
    """The whole filtered distribution q at BASELINE's full vocabulary for top-p-only rows (the exact
    cluster kernel: float64 bucket masses, boundary walk) and a min-p-only row, vs the oracle's q."""
    wl = make_workload("c2", B=3)
    wl.params[2] = RowParams(temperature=0.8, min_p=0.01, seed=5, request_id=5)
    orc = oracle_run(wl, step=3, want_q=True)
    s, out = _run(wl, step=3, q=True)
    assert_parity(wl, out, orc, q=out["q"])


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_exact_kernel_near_tie_floods(dtype):
    """Rows whose boundary (sub-)bucket holds far more than the exact kernel's 4096-entry gather buffer:
    all-equal rows (top-p-only, top-k 3000 > K_cand, min-p), a two-valued row and a ramp of values
    closer than 1/65536 octave of weight — resolved by the composite radix rounds, vs the oracle's q."""
    B, V = 7, 60000
    z = np.full((B, V), 0.75, dtype=np.float32)
    z[6] = -np.arange(V, dtype=np.float32) * np.float32(0.02)   # top_k's cutoff deep in the far-tail bucket
    z[3, ::2] = np.float32(0.5)
    z[4] = (np.float32(1.0) + np.arange(V, dtype=np.float32) * np.float32(2 ** -23)).astype(np.float32)
    z[5, 1000:] = np.float32(-np.inf)
    if dtype == "bf16":
        from workloads.synth import f32_to_bf16_bits
        raw = f32_to_bf16_bits(z)
    else:
        raw = z
    params = [RowParams(temperature=1.0, top_p=0.5, seed=1, request_id=1),
              RowParams(temperature=0.7, top_k=3000, seed=2, request_id=2),
              RowParams(temperature=1.0, top_k=5000, top_p=0.3, seed=3, request_id=3),
              RowParams(temperature=1.0, top_p=0.9, seed=4, request_id=4),
              RowParams(temperature=1.0, top_p=0.77, seed=5, request_id=5),
              RowParams(temperature=1.0, top_p=0.6, seed=6, request_id=6),
              RowParams(temperature=1.0, top_k=5000, seed=7, request_id=7)]
    wl = Workload("ties", B, V, dtype, raw, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=1, want_q=True)
    s, out = _run(wl, step=1, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s, out = _run(wl, step=1)
    assert_parity(wl, out, oracle_run(wl, 1))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_extreme_magnitudes_and_param_edges(dtype):
    """Logits near the binary32 / bf16 range limits (differences overflow to inf in binary32, weights
    underflow to 0 in float64), huge temperatures, min_p = 1, top_p at the smallest float, top_k = V - 1."""
    B, V = 10, 7000
    rng = np.random.default_rng(5)
    z = rng.normal(0, 3, size=(B, V)).astype(np.float32)
    z[0, 10] = np.float32(3e38)
    z[0, 20] = np.float32(-3e38)
    z[1] = (rng.normal(0, 1, size=V) * 1e30).astype(np.float32)
    z[2, ::3] = np.float32(-3e38)
    z[3] = np.float32(1e20)
    z[3, 5::7] = np.float32(1e20 * (1 + 2 ** -6))
    z[4, :] = np.float32(-1e35)
    z[4, 6999] = np.float32(-9e34)
    if dtype == "bf16":
        from workloads.synth import f32_to_bf16_bits
        raw = f32_to_bf16_bits(z)
    else:
        raw = z
    params = [RowParams(temperature=1.0, top_p=0.9, seed=0, request_id=0),
              RowParams(temperature=1e30, top_k=300, seed=1, request_id=1),
              RowParams(temperature=2.0, min_p=0.5, seed=2, request_id=2),
              RowParams(temperature=1e19, top_p=0.5, seed=3, request_id=3),
              RowParams(temperature=1e33, seed=4, request_id=4),
              RowParams(temperature=0.9, min_p=1.0, seed=5, request_id=5),
              RowParams(temperature=1.0, top_p=float(np.float32(1e-38)), seed=6, request_id=6),
              RowParams(temperature=0.6, top_k=V - 1, seed=7, request_id=7),
              RowParams(temperature=3e38, top_k=V - 1, top_p=0.999, seed=8, request_id=8),
              RowParams(temperature=1.0, top_k=1, min_p=0.9, seed=9, request_id=9)]
    wl = Workload("extreme", B, V, dtype, raw, [[]] * B, [[]] * B, params)
    orc = oracle_run(wl, step=6, want_q=True)
    s, out = _run(wl, step=6, q=True)
    assert_parity(wl, out, orc, q=out["q"])
    s, out = _run(wl, step=6)
    assert_parity(wl, out, oracle_run(wl, 6))


@pytest.mark.parametrize("cfg,dtype,V", [("c2", "f32", None), ("c4", "f32", None), ("c3", "f32", None),
                                         ("c2", "bf16", 262144), ("c4", "bf16", 256000)])
def test_dtype_and_vocabulary_variants(cfg, dtype, V):
    """Binary32 logits at the configs' full vocabularies (the exact kernel's per-element path for the
    unbounded rows) and 256K-class vocabularies in bf16 (more CTAs per row in the exact kernel)."""
    wl = make_workload(cfg, B=8, V=V, dtype=dtype)
    s, out = _run(wl, step=2)
    assert_parity(wl, out, oracle_run(wl, 2))


def test_history_append_through_exact_kernel_rows():
    """Decode steps of top-p-only rows (appended by the exact cluster kernel) and mixed c4 rows, against
    the oracle replaying the grown histories; the incremental tables equal a recount."""
    import torch
    for cfg, B in (("c2", 6), ("c4", 9)):
        wl = make_workload(cfg, B=B)
        s = make_sampler(wl, max_history=2400)
        x = device_logits(wl)
        outputs = [list(o) for o in wl.outputs]
        for step in range(4):
            out = s.sample(x, step, append=True)
            torch.cuda.synchronize()
            cur = Workload(wl.name, wl.B, wl.V, wl.dtype, wl.raw, wl.prompts, [list(o) for o in outputs], wl.params)
            assert_parity(cur, out, oracle_run(cur, step))
            for b, t in enumerate(out["tokens"].cpu().tolist()):
                outputs[b].append(int(t))
        for b in range(wl.B):
            h = s.get_history(b)
            assert h["output"] == outputs[b]
            ids = sorted(set(wl.prompts[b]) | set(outputs[b]))
            assert h["uniq_ids"] == ids
            assert h["uniq_counts"] == [outputs[b].count(i) for i in ids]


@pytest.mark.parametrize("cfg", ["c3", "c2"])
def test_graph_replays_advance_a_device_step(cfg):
    """A decode step captured ONCE (sample with in-kernel append + the step increment) and replayed: with
    sampler_set_step_source every replay draws with the next Philox step (TSEM-style versioned per-step
    input) and equals eager sampling with host steps, append included (c2: exact-kernel rows)."""
    import torch
    wl = make_workload(cfg, B=8, V=20000)
    x = device_logits(wl)
    ref = make_sampler(wl, max_history=1024)
    s = make_sampler(wl, max_history=1024)
    step = torch.tensor([100], dtype=torch.int64, device="cuda")
    s.set_step_source(step)
    out = s._outs(wl.B, None)
    s.sample(x, 0, out=out)  # warm-up (no append)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        s.sample(x, 0, out=out, append=True)
        step.add_(1)
    toks = []
    for i in range(4):
        g.replay()
        r = ref.sample(x, 100 + i, append=True)
        torch.cuda.synchronize()
        assert torch.equal(out["tokens"], r["tokens"]), i
        assert torch.allclose(out["logprobs"], r["logprobs"], rtol=1e-6, atol=1e-7)
        toks.append(out["tokens"].clone())
    assert any(not torch.equal(toks[0], t) for t in toks[1:])  # the draws moved with the step
    assert int(step.item()) == 104
    for b in range(wl.B):
        assert s.get_history(b)["output"] == ref.get_history(b)["output"]
    s.set_step_source(None)

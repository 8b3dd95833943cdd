"""Host-side logic of the N>1 paths, on CPU with the gloo backend, world_size 2.

* vocab sharding (TP lm_head style): the shard bounds tile [0, V) and every rank
  receives every rank's candidate record, in rank order, from ONE all_gather_into_tensor —
  checked through paper_2506_22033_b200.distributed.sample_vocab_sharded with a stand-in sampler
  object (the CUDA kernels behind sample_local / merge are covered by the -m gpu tests, including
  the sharded == unsharded parity with an in-process gather);
* batch-row sharding (DP style): the row bounds tile [0, B) with no collective on the data path;
* bench.py's max-over-ranks reduction of the timed region.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_22033_b200.distributed import (batch_row_bounds, sample_batch_sharded, sample_vocab_sharded,
                                               setup_peer_exchange, vocab_shard_bounds)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("V", [32000, 128256, 129280, 152064, 7, 8])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_vocab_shard_bounds_tile_the_vocabulary(V, world):
    prev = 0
    for r in range(world):
        lo, hi = vocab_shard_bounds(V, world, r)
        assert lo == prev and hi >= lo
        if hi < V:
            assert (hi - lo) % 8 == 0  # 16-byte bf16 rows in every shard but the last
        prev = hi
    assert prev == V


@pytest.mark.parametrize("B", [1, 3, 256, 1024])
@pytest.mark.parametrize("world", [1, 2, 8])
def test_batch_row_bounds_tile_the_batch(B, world):
    prev = 0
    for r in range(world):
        lo, hi = batch_row_bounds(B, world, r)
        assert lo == prev
        prev = hi
    assert prev == B


class _StandInSampler:
    """Plays the C-ABI handle's part in the exchange: record = (rank, row, byte index) pattern."""

    def __init__(self, rank, rec_bytes_per_row):
        self.rank, self.rb = rank, rec_bytes_per_row
        self.merged = None

    def record_bytes(self, B):
        return self.rb * B

    def sample_local(self, logits_slice, rec, slots=None, params=None):
        B = logits_slice.shape[0]
        v = torch.arange(self.rb * B, dtype=torch.int64)
        rec.copy_(((v + 31 * self.rank + 7) % 251).to(torch.uint8))

    def merge(self, gathered, world, B, step, slots=None, params=None, seeds=None, append=False, out=None):
        self.merged = (gathered.clone(), world, B, step)
        return {"tokens": torch.zeros(B, dtype=torch.int32)}

    # NEXT-2: exchange buffer handles (64 bytes, rank-specific) and the peer mapping call
    def exchange_init(self, world, rank, timeout_ms=0):
        return bytes([rank + 1]) * 64, 0x1000 * (rank + 1)

    def exchange_open(self, handles):
        self.opened = handles

    # NEXT-1 resolve rounds: payload = (rank, round) pattern; 3 rounds of work, then no row is active
    def resolve_bytes(self, B):
        return 16 * B

    def resolve_round(self, logits_slice, step, rnd, gathered, world, rank, payload, out, slots=None, params=None,
                      seeds=None, append=False, active=None, stream=None):
        if rnd > 0:
            pb = payload.numel()
            ok = all(torch.equal(gathered[r * pb:(r + 1) * pb], torch.full((pb,), 16 * r + rnd - 1, dtype=torch.uint8))
                     for r in range(world))
            self.rounds_ok = getattr(self, "rounds_ok", True) and ok
        self.last_round = rnd
        payload.fill_(16 * rank + rnd)
        active.fill_(max(0, 3 - rnd))

    def sample(self, logits_rows, step, slots=None, params=None, seeds=None, append=False, out=None):
        # stand-in result: token = 1000 * rank + local row, logprob = -(token) / 8
        n = logits_rows.shape[0]
        tok = (1000 * self.rank + torch.arange(n)).to(torch.int32)
        return {"tokens": tok, "logprobs": -tok.to(torch.float32) / 8}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, V = 5, 1000
        lo, hi = vocab_shard_bounds(V, world, rank)
        s = _StandInSampler(rank, rec_bytes_per_row=48 + 8 * 40)
        out = sample_vocab_sharded(s, torch.zeros(B, hi - lo), step=3)
        g, w, b, step = s.merged
        ok = w == world and b == B and step == 3 and "tokens" in out
        ok = ok and s.rounds_ok and s.last_round == 3  # adaptive stop: 3 exchanges, rank-ordered payloads
        # the fixed round count (CUDA-graph mode): exactly `rounds` exchanges whatever the active count
        from paper_2506_22033_b200.distributed import resolve_unbounded
        s.rounds_ok = True
        n = resolve_unbounded(s, torch.zeros(B, hi - lo), 4, {}, lambda g, p: dist.all_gather_into_tensor(g, p),
                              world, rank, rounds=5)
        ok = ok and n == 5 and s.last_round == 5
        rb = s.record_bytes(B)
        for r in range(world):
            v = torch.arange(rb, dtype=torch.int64)
            ok = ok and torch.equal(g[r * rb:(r + 1) * rb], ((v + 31 * r + 7) % 251).to(torch.uint8))
        # NEXT-2: every rank maps every rank's exchange buffer from the handles, in rank order
        setup_peer_exchange(s)
        ok = ok and s.opened == b"".join(bytes([r + 1]) * 64 for r in range(world))
        # batch-row sharding of one global batch of 7 rows: every rank ends with the whole result
        Bg = 7
        blo, bhi = batch_row_bounds(Bg, world, rank)
        o = sample_batch_sharded(s, torch.zeros(bhi - blo, 4), step=1, B_global=Bg)
        exp_tok = []
        for r in range(world):
            l2, h2 = batch_row_bounds(Bg, world, r)
            exp_tok += [1000 * r + i for i in range(h2 - l2)]
        ok = ok and o["tokens"].tolist() == exp_tok
        ok = ok and torch.equal(o["logprobs"], -torch.tensor(exp_tok, dtype=torch.float32) / 8)
        # bench.py: time of the slowest rank
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = ok and float(t.item()) == float(world)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_vocab_sharded_exchange_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}

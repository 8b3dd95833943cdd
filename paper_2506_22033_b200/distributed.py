"""Multi-GPU glue over torch.distributed (NCCL over NVLink 5 / NVSwitch): plumbing only.

Two shardings of the sampling task:
  * vocab-sharded (TP lm_head style; the paper's B x V/t logits shards): each rank reduces
    its slice to per-row candidate records (sampler_sample_local), ONE all_gather_into_tensor of
    those few-KB records, then every rank runs the same deterministic merge (sampler_merge).
  * batch-row sharded (DP style, P:24 footnote): each rank samples its own rows, no collective on the
    data path; optionally one all-gather of the sampled tokens / logprobs (8 B per row) so that every
    rank holds the whole batch's result.
Both are capturable in a CUDA graph (pass preallocated `rec` / `gathered` / `out` buffers).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .sampler import Sampler


def vocab_shard_bounds(V: int, world: int, rank: int, align: int = 8):
    """Contiguous slices, each a multiple of `align` ids except possibly the last."""
    per = -(-V // world)
    per = -(-per // align) * align
    lo = min(V, rank * per)
    hi = min(V, lo + per)
    return lo, hi


def sample_vocab_sharded(sampler: Sampler, logits_slice: torch.Tensor, step: int, group=None,
                         slots=None, params=None, seeds=None, append=False, rec=None, gathered=None, out=None,
                         resolve=True, resolve_rounds=None, resolve_bufs=None):
    """Two-phase vocab-sharded sampling over a torch.distributed process group (NCCL): local candidate
    records -> ONE all_gather_into_tensor (rank order) -> the same deterministic merge on every rank.
    Rows the candidates do not bound (top-p-only / min-p-only / unfiltered, top_k > max_top_k) are then
    finished by the resolve rounds (NEXT-1, `resolve_unbounded`) unless resolve=False.
    With rec / gathered / out / resolve_bufs preallocated the call allocates nothing; under CUDA-graph
    capture the resolve round count defaults to its bound (resolve_max_rounds), so it never synchronises.
    A caller whose rows are all bounded by top_k <= max_top_k (or greedy) passes resolve=False."""
    B = logits_slice.shape[0]
    rb = sampler.record_bytes(B)
    world = dist.get_world_size(group)
    if rec is None:
        rec = torch.empty(rb, dtype=torch.uint8, device=logits_slice.device)
    if gathered is None:
        gathered = torch.empty(world * rb, dtype=torch.uint8, device=logits_slice.device)
    sampler.sample_local(logits_slice, rec, slots=slots, params=params)
    dist.all_gather_into_tensor(gathered, rec, group=group)
    out = sampler.merge(gathered, world, B, step, slots=slots, params=params, seeds=seeds, append=append, out=out)
    if resolve:
        if resolve_rounds is None and logits_slice.is_cuda and torch.cuda.is_current_stream_capturing():
            resolve_rounds = sampler.resolve_max_rounds()  # no host read inside a graph: the bound
        resolve_unbounded(sampler, logits_slice, step, out, lambda g, p: dist.all_gather_into_tensor(g, p, group=group),
                          world, dist.get_rank(group), slots=slots, params=params, seeds=seeds, append=append,
                          rounds=resolve_rounds, bufs=resolve_bufs)
    return out


def setup_peer_exchange(sampler: Sampler, group=None, timeout_ms=0):
    """NEXT-2 plumbing: allocate this rank's exchange buffer, all-gather the 64-byte CUDA IPC handles
    (rank order) over the process group, map every peer's buffer (sampler_exchange_open)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    h, _ = sampler.exchange_init(world, rank, timeout_ms)
    allh = [None] * world
    dist.all_gather_object(allh, h, group=group)
    sampler.exchange_open(b"".join(allh))
    return allh


def sample_vocab_sharded_p2p(sampler: Sampler, logits_slice: torch.Tensor, step: int, group=None, slots=None,
                             params=None, seeds=None, append=False, out=None, resolve=False, resolve_rounds=None,
                             resolve_bufs=None):
    """The vocab-sharded step through the one-shot peer exchange (after setup_peer_exchange): one library call
    for the candidate step and, with resolve=True, the resolve rounds for rows the candidates do not bound,
    their payloads also through the peer exchange — no collective call on the data path.  resolve_rounds:
    None = adaptive (one 4-byte read per round; under graph capture the bound), or a fixed count."""
    out = sampler.sample_exchange(logits_slice, step, slots=slots, params=params, seeds=seeds, append=append,
                                  out=out)
    if resolve:
        if resolve_rounds is None and logits_slice.is_cuda and torch.cuda.is_current_stream_capturing():
            resolve_rounds = sampler.resolve_max_rounds()
        active = resolve_bufs[2] if resolve_bufs is not None else torch.zeros(1, dtype=torch.int32,
                                                                              device=logits_slice.device)
        kw = dict(slots=slots, params=params, seeds=seeds, append=append, active=active)
        sampler.resolve_round_exchange(logits_slice, step, 0, out, **kw)
        n = 0
        while (resolve_rounds is None and int(active.item()) > 0) or (resolve_rounds is not None and n < resolve_rounds):
            n += 1
            sampler.resolve_round_exchange(logits_slice, step, n, out, **kw)
    return out


def resolve_buffers(sampler: Sampler, B: int, world: int, device):
    """(payload, gathered, active) buffers for resolve_unbounded."""
    nb = sampler.resolve_bytes(B)
    return (torch.empty(nb, dtype=torch.uint8, device=device), torch.empty(world * nb, dtype=torch.uint8, device=device),
            torch.zeros(1, dtype=torch.int32, device=device))


def resolve_unbounded(sampler: Sampler, logits_slice: torch.Tensor, step: int, out: dict, exchange, world: int,
                      rank: int, slots=None, params=None, seeds=None, append=False, rounds=None, bufs=None):
    """NEXT-1: finish the rows sampler_merge left SAMPLER_ROW_UNRESOLVED (include/sampler.h, resolve rounds).
    exchange(gathered, payload) must all-gather the ranks' payloads in rank order (NCCL all_gather_into_tensor).
    rounds=None: stop as soon as no row is active (one 4-byte device->host read per round); an int: exactly
    that many exchanges (sampler.resolve_max_rounds() always suffices; CUDA-graph capturable).
    Returns the number of exchanges issued."""
    B = logits_slice.shape[0]
    payload, gathered, active = bufs if bufs is not None else resolve_buffers(sampler, B, world, logits_slice.device)
    kw = dict(slots=slots, params=params, seeds=seeds, append=append, active=active)
    sampler.resolve_round(logits_slice, step, 0, None, world, rank, payload, out, **kw)
    n = 0
    while (rounds is None and int(active.item()) > 0) or (rounds is not None and n < rounds):
        exchange(gathered, payload)
        n += 1
        sampler.resolve_round(logits_slice, step, n, gathered, world, rank, payload, out, **kw)
    return n


def batch_row_bounds(B: int, world: int, rank: int):
    per = -(-B // world)
    lo = min(B, rank * per)
    return lo, min(B, lo + per)


def sample_batch_sharded(sampler: Sampler, logits_rows: torch.Tensor, step: int, B_global: int, group=None,
                         slots=None, params=None, seeds=None, append=False, out=None, gather=True):
    """Batch-row sharding (DP style): this rank samples its rows [lo, hi) = batch_row_bounds(B_global,
    world, rank) with no collective on the data path; with gather=True one all-gather of the
    (token, logprob) pairs returns the whole batch's result on every rank (rows in global order)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = batch_row_bounds(B_global, world, rank)
    assert logits_rows.shape[0] == hi - lo
    o = sampler.sample(logits_rows, step, slots=slots, params=params, seeds=seeds, append=append, out=out)
    if not gather:
        return o
    per = -(-B_global // world)
    dev = logits_rows.device
    pair = torch.full((per, 2), -1, dtype=torch.int32, device=dev)
    pair[: hi - lo, 0] = o["tokens"]
    pair[: hi - lo, 1] = o["logprobs"].view(torch.int32)
    allp = torch.empty((world * per, 2), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(allp, pair, group=group)
    allp = allp[:B_global]
    return dict(tokens=allp[:, 0].contiguous(), logprobs=allp[:, 1].contiguous().view(torch.float32), local=o)

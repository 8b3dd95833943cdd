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
                         slots=None, params=None, seeds=None, append=False, rec=None, gathered=None, out=None):
    """Two-phase vocab-sharded sampling over a torch.distributed process group (NCCL): local candidate
    records -> ONE all_gather_into_tensor (rank order) -> the same deterministic merge on every rank.
    With rec / gathered / out preallocated the call allocates nothing (CUDA-graph capturable)."""
    B = logits_slice.shape[0]
    rb = sampler.record_bytes(B)
    world = dist.get_world_size(group)
    if rec is None:
        rec = torch.empty(rb, dtype=torch.uint8, device=logits_slice.device)
    if gathered is None:
        gathered = torch.empty(world * rb, dtype=torch.uint8, device=logits_slice.device)
    sampler.sample_local(logits_slice, rec, slots=slots, params=params)
    dist.all_gather_into_tensor(gathered, rec, group=group)
    return sampler.merge(gathered, world, B, step, slots=slots, params=params, seeds=seeds, append=append, out=out)


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

"""Multi-GPU glue over torch.distributed (NCCL over NVLink 5 / NVSwitch): plumbing only.

Two shardings of the sampling task:
  * vocab-sharded (TP lm_head style; the paper's B x V/t logits shards): each rank reduces
    its slice to per-row candidate records (sampler_sample_local), ONE all_gather_into_tensor of
    those few-KB records, then every rank runs the same deterministic merge (sampler_merge).
  * batch-row sharded (DP style, P:24 footnote): each rank samples its own rows, no collective.
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
                         slots=None, params=None, seeds=None, append=False):
    """Two-phase vocab-sharded sampling over a torch.distributed process group (NCCL)."""
    B = logits_slice.shape[0]
    rb = sampler.record_bytes(B)
    world = dist.get_world_size(group)
    rec = torch.empty(rb, dtype=torch.uint8, device=logits_slice.device)
    sampler.sample_local(logits_slice, rec, slots=slots, params=params)
    gathered = torch.empty(world * rb, dtype=torch.uint8, device=logits_slice.device)
    dist.all_gather_into_tensor(gathered, rec, group=group)
    return sampler.merge(gathered, world, B, step, slots=slots, params=params, seeds=seeds, append=append)


def batch_row_bounds(B: int, world: int, rank: int):
    per = -(-B // world)
    lo = min(B, rank * per)
    return lo, min(B, lo + per)

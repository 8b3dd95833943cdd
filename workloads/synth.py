"""Seeded synthetic workloads shared by tests, bench.py and smoke().

This module holds NO arithmetic of the sampling method: it only draws random
logits, histories and per-row parameters with the shapes/value structure of the
paper's workloads (DESIGN.md §4 "input recipe", = SURVEY.md §8(d)), so that the
oracle and the CUDA path are fed identical inputs.

Logits (per row):
  * z = 2.0*N(0,1); a "head" of 16 random ids gets +U(4,12)  (a peaked LLM-like row)
  * a quarter of the rows are "flat": z = N(0,1), no head (large top-p nuclei)
  * 1% of rows get an exact duplicate of the row max at another id (tie tests)
  * cast to the config dtype with round-to-nearest-even
Histories: prompt + output token lists; half the tokens drawn from the row's
top-200 logit ids (so penalties change outcomes), half Zipf(1.2) over a per-row
permutation of the vocabulary (repeats; counts up to ~20).
The paper's real ShareGPT logits are unavailable: stand-in only.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 20250627


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round-to-nearest-even; NaN kept NaN."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if np.any(nan):
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


@dataclass
class RowParams:
    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0
    min_p: float = 0.0
    repetition_penalty: float = 1.0
    presence_penalty: float = 0.0
    frequency_penalty: float = 0.0
    seed: int = 0
    request_id: int = 0


@dataclass
class Workload:
    name: str
    B: int
    V: int
    dtype: str                      # 'bf16' | 'f32'
    raw: np.ndarray                 # [B, V] uint16 (bf16 bits) or float32
    prompts: list = field(default_factory=list)
    outputs: list = field(default_factory=list)
    params: list = field(default_factory=list)

    def logits_f32(self) -> np.ndarray:
        return bf16_bits_to_f32(self.raw) if self.dtype == "bf16" else self.raw


def gen_logits(rng: np.random.Generator, B: int, V: int, dtype: str,
               flat_frac: float = 0.25, tie_frac: float = 0.01, head: int = 16):
    z = np.empty((B, V), dtype=np.float32)
    for b in range(B):
        flat = rng.random() < flat_frac
        if flat:
            row = rng.standard_normal(V, dtype=np.float32)
        else:
            row = 2.0 * rng.standard_normal(V, dtype=np.float32)
            ids = rng.choice(V, size=min(head, V), replace=False)
            row[ids] += rng.uniform(4.0, 12.0, size=len(ids)).astype(np.float32)
        if rng.random() < tie_frac and V > 1:
            m = int(np.argmax(row))
            other = int(rng.integers(0, V))
            if other != m:
                row[other] = row[m]
        z[b] = row
    if dtype == "bf16":
        raw = f32_to_bf16_bits(z)
        # keep injected ties exact after rounding (both copies round identically)
        return raw
    return z


def gen_history(rng: np.random.Generator, raw_row_f32: np.ndarray, n_prompt: int, n_output: int,
                top_pool: int = 200, zipf_a: float = 1.2):
    V = len(raw_row_f32)
    n = n_prompt + n_output
    if n == 0:
        return [], []
    pool = np.argpartition(-raw_row_f32, min(top_pool, V) - 1)[:min(top_pool, V)]
    perm = rng.permutation(V)
    toks = np.empty(n, dtype=np.int64)
    from_pool = rng.random(n) < 0.5
    toks[from_pool] = rng.choice(pool, size=int(from_pool.sum()))
    nz = int((~from_pool).sum())
    if nz:
        zr = rng.zipf(zipf_a, size=nz)
        zr = np.minimum(zr - 1, V - 1)
        toks[~from_pool] = perm[zr]
    toks = toks.astype(np.int32)
    return toks[:n_prompt].tolist(), toks[n_prompt:].tolist()


# ----------------------------------------------------------------- configs (BASELINE.json)
CONFIGS = {
    # configs[0]: B=4, V=32000 fp32, greedy + temperature 0.8 top-k=50 top-p=0.9, fixed seed
    "c1": dict(B=4, V=32000, dtype="f32"),
    # configs[1]: Llama-3-8B-shaped B=64, V=128256 bf16, top-p=0.95 + rep/pres/freq over 512-token hist
    "c2": dict(B=64, V=128256, dtype="bf16"),
    # configs[2]: Qwen2.5-72B-shaped B=256, V=152064 bf16, top-k=40 top-p=0.9 min-p=0.05 + penalties
    "c3": dict(B=256, V=152064, dtype="bf16"),
    # configs[3]: DeepSeek-V3-shaped B=1024, V=129280 bf16, mixed per-row params
    "c4": dict(B=1024, V=129280, dtype="bf16"),
    # configs[4]: latency sweep B=1..32, V=152064
    "c5": dict(B=32, V=152064, dtype="bf16"),
}


def row_params(cfg: str, b: int, run: int = 0) -> RowParams:
    req = b + (run << 32)
    if cfg == "c1":
        if b < 2:
            return RowParams(temperature=0.0, seed=1234 + b, request_id=req)
        return RowParams(temperature=0.8, top_k=50, top_p=0.9, seed=1234 + b, request_id=req)
    if cfg == "c2":
        return RowParams(temperature=1.0, top_p=0.95, repetition_penalty=1.1,
                         presence_penalty=0.4, frequency_penalty=0.3, seed=7 + b, request_id=req)
    if cfg in ("c3", "c5"):
        return RowParams(temperature=0.7, top_k=40, top_p=0.9, min_p=0.05, repetition_penalty=1.1,
                         presence_penalty=0.4, frequency_penalty=0.3, seed=11 + b, request_id=req)
    if cfg == "c4":
        pen = (b % 2 == 0)
        kw = dict(repetition_penalty=1.1, presence_penalty=0.4, frequency_penalty=0.3) if pen else {}
        m = b % 3
        if m == 0:
            return RowParams(temperature=0.0, seed=5 + b, request_id=req, **kw)
        if m == 1:
            return RowParams(temperature=0.8, top_k=[20, 50, 100][(b // 3) % 3], seed=5 + b,
                             request_id=req, **kw)
        return RowParams(temperature=1.0, top_p=[0.8, 0.9, 0.95][(b // 3) % 3], seed=5 + b,
                         request_id=req, **kw)
    raise KeyError(cfg)


def history_lengths(cfg: str, rng: np.random.Generator):
    if cfg in ("c2", "c3", "c5"):
        return 384, 128
    if cfg == "c4":
        n = int(rng.integers(0, 2049))
        npr = int(rng.integers(0, n + 1))
        return npr, n - npr
    return 0, 0


def make_workload(cfg: str, B: int | None = None, V: int | None = None, seed_offset: int = 0,
                  run: int = 0, with_history: bool = True, dtype: str | None = None) -> Workload:
    """Build the seeded workload of config `cfg` (optionally resized for parity tests)."""
    base = CONFIGS[cfg]
    B = base["B"] if B is None else B
    V = base["V"] if V is None else V
    dtype = base["dtype"] if dtype is None else dtype
    idx = list(CONFIGS).index(cfg)
    rng = np.random.default_rng(BASE_SEED + idx + 1000 * seed_offset)
    raw = gen_logits(rng, B, V, dtype)
    f = bf16_bits_to_f32(raw) if dtype == "bf16" else raw
    prompts, outputs = [], []
    for b in range(B):
        npr, nout = history_lengths(cfg, rng) if with_history else (0, 0)
        p, o = gen_history(rng, f[b], npr, nout)
        prompts.append(p)
        outputs.append(o)
    params = [row_params(cfg, b, run) for b in range(B)]
    return Workload(cfg, B, V, dtype, raw, prompts, outputs, params)


def random_params(rng: np.random.Generator, b: int, V: int) -> RowParams:
    """Random mixed per-row params for property/parity sweeps."""
    kind = int(rng.integers(0, 6))
    t = [0.0, 0.5, 0.7, 1.0, 1.3][int(rng.integers(0, 5))]
    p = RowParams(temperature=t, seed=int(rng.integers(0, 2**63)), request_id=int(rng.integers(0, 2**63)))
    if kind in (1, 4, 5):
        p.top_k = int(rng.integers(1, min(V, 300) + 1))
    if kind in (2, 4, 5):
        p.top_p = float(rng.choice([0.5, 0.8, 0.9, 0.95, 0.99]))
    if kind in (3, 5):
        p.min_p = float(rng.choice([0.01, 0.05, 0.1, 0.3]))
    if rng.random() < 0.5:
        p.repetition_penalty = float(rng.choice([0.8, 1.1, 1.3]))
        p.presence_penalty = float(rng.choice([0.0, 0.4, -0.2]))
        p.frequency_penalty = float(rng.choice([0.0, 0.3, 0.05]))
    return p


def device_logits(wl: Workload, ld=None, device="cuda"):
    """The workload's logits as a torch CUDA tensor [B, V] (row stride ld >= V when given).
    Placement only (no arithmetic of the method); used by tests, smoke() and bench.py."""
    import torch
    ld = wl.V if ld is None else ld
    if wl.dtype == "bf16":
        buf = np.zeros((wl.B, ld), dtype=np.uint16)
        buf[:, :wl.V] = wl.raw
        t = torch.from_numpy(buf.view(np.int16)).view(torch.bfloat16)
    else:
        buf = np.zeros((wl.B, ld), dtype=np.float32)
        buf[:, :wl.V] = wl.raw
        t = torch.from_numpy(buf)
    t = t.to(device)
    return t[:, :wl.V] if ld != wl.V else t

"""Thin Python binding over the C ABI (include/sampler.h) — argument marshalling only.

Every step of the sampling path runs in the sm_100a kernels of libsampler_b200.so; PyTorch is
used only for device memory and streams.  There is no CPU fallback: if the library is missing
this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsampler_b200.so")

SAMPLER_OK, SAMPLER_EINVAL, SAMPLER_ENOMEM, SAMPLER_ECUDA, SAMPLER_ERANGE, SAMPLER_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
SAMPLER_F32, SAMPLER_BF16 = 0, 2
PEN_OPENAI_CTRL, PEN_LINEAR = 0, 1
ROW_OK, ROW_NONFINITE, ROW_ALL_NEG_INF, ROW_UNRESOLVED, ROW_INVALID, ROW_EXCHANGE_TIMEOUT = 0, 1, 2, 3, 4, 5

EXPORTED = [
    "sampler_create", "sampler_destroy", "sampler_last_error", "sampler_set_params", "sampler_set_history",
    "sampler_append_tokens", "sampler_get_history", "sampler_sample", "sampler_debug_distribution",
    "sampler_record_bytes", "sampler_sample_local", "sampler_merge", "sampler_last_launch_count",
    "sampler_version", "sampler_debug_trace", "sampler_set_timing", "sampler_kernel_times",
    "sampler_resolve_bytes", "sampler_resolve_round", "sampler_resolve_max_rounds",
    "sampler_exchange_init", "sampler_exchange_open", "sampler_exchange_set_peers", "sampler_sample_exchange",
    "sampler_get_slot_flags", "sampler_set_step_source", "sampler_resolve_round_exchange",
]


class SamplerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"sampler error {code}: {msg}")
        self.code = code


class CConfig(C.Structure):
    _fields_ = [("vocab_size", C.c_int32), ("vocab_offset", C.c_int32), ("vocab_local", C.c_int32),
                ("max_batch", C.c_int32), ("max_history", C.c_int32), ("max_top_k", C.c_int32),
                ("logits_dtype", C.c_int32), ("penalty_mode", C.c_int32), ("device", C.c_int32)]


class CParams(C.Structure):
    _fields_ = [("temperature", C.c_float), ("top_k", C.c_int32), ("top_p", C.c_float), ("min_p", C.c_float),
                ("repetition_penalty", C.c_float), ("presence_penalty", C.c_float),
                ("frequency_penalty", C.c_float), ("reserved", C.c_int32), ("seed", C.c_uint64),
                ("request_id", C.c_uint64)]


assert C.sizeof(CParams) == 48

PARAMS_DTYPE = np.dtype([("temperature", "<f4"), ("top_k", "<i4"), ("top_p", "<f4"), ("min_p", "<f4"),
                         ("repetition_penalty", "<f4"), ("presence_penalty", "<f4"),
                         ("frequency_penalty", "<f4"), ("reserved", "<i4"), ("seed", "<u8"),
                         ("request_id", "<u8")])
assert PARAMS_DTYPE.itemsize == 48


@dataclass
class SamplingParams:
    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0
    min_p: float = 0.0
    repetition_penalty: float = 1.0
    presence_penalty: float = 0.0
    frequency_penalty: float = 0.0
    seed: int = 0
    request_id: int = 0


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2506_22033_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "sampler_create": ([C.POINTER(CConfig), C.POINTER(P)], I32),
        "sampler_destroy": ([P], I32),
        "sampler_last_error": ([P], C.c_char_p),
        "sampler_set_params": ([P, I32, P, P], I32),
        "sampler_set_history": ([P, I32, P, I32, P, I32], I32),
        "sampler_append_tokens": ([P, I32, P, P], I32),
        "sampler_get_history": ([P, I32, P, P, P, P, P, P, P, P], I32),
        "sampler_sample": ([P, P, I64, I32, P, P, P, U64, I32, P, P, P, P, P], I32),
        "sampler_debug_distribution": ([P, P, I64, I32, P, P, P, U64, P, P, P, P], I32),
        "sampler_record_bytes": ([P, I32], I64),
        "sampler_sample_local": ([P, P, I64, I32, P, P, P, P], I32),
        "sampler_merge": ([P, P, I32, I32, P, P, P, U64, I32, P, P, P, P, P], I32),
        "sampler_resolve_bytes": ([P, I32], I64),
        "sampler_resolve_round": ([P, P, I64, I32, P, P, P, U64, I32, P, I32, I32, P, I32, P, P, P, P, P, P], I32),
        "sampler_resolve_max_rounds": ([], I32),
        "sampler_exchange_init": ([P, I32, I32, C.c_uint32, P, P], I32),
        "sampler_exchange_open": ([P, P], I32),
        "sampler_get_slot_flags": ([P, I32, P], I32),
        "sampler_set_step_source": ([P, P], I32),
        "sampler_resolve_round_exchange": ([P, P, I64, I32, P, P, P, U64, I32, I32, P, P, P, P, P, P], I32),
        "sampler_exchange_set_peers": ([P, P], I32),
        "sampler_sample_exchange": ([P, P, I64, I32, P, P, P, U64, I32, P, P, P, P, I32, P], I32),
        "sampler_last_launch_count": ([P], I32),
        "sampler_version": ([], C.c_char_p),
        "sampler_debug_trace": ([P, P, I32], I32),
        "sampler_set_timing": ([P, I32], I32),
        "sampler_kernel_times": ([P, P, I32, P], I32),
    }
    for name, (argt, rest) in sig.items():
        f = getattr(lib, name)
        f.argtypes = argt
        f.restype = rest
    return lib


_lib = _load()


def lib():
    return _lib


def version() -> str:
    return _lib.sampler_version().decode()


def pack_params(params) -> np.ndarray:
    """list of SamplingParams / dicts / objects with the same attributes -> structured array."""
    arr = np.zeros(len(params), dtype=PARAMS_DTYPE)
    for i, p in enumerate(params):
        for f in fields(SamplingParams):
            v = p[f.name] if isinstance(p, dict) else getattr(p, f.name)
            if f.name in ("seed", "request_id"):
                v = int(v) & 0xFFFFFFFFFFFFFFFF
            arr[i][f.name] = v
    return arr


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Sampler:
    """One handle over the C ABI.  Tensors are torch CUDA tensors on the handle's device."""

    def __init__(self, vocab_size, max_batch, max_history=4096, max_top_k=128, dtype="bf16",
                 penalty_mode=PEN_OPENAI_CTRL, device=0, vocab_offset=0, vocab_local=None):
        cfg = CConfig(vocab_size, vocab_offset, vocab_size if vocab_local is None else vocab_local, max_batch,
                      max_history, max_top_k, SAMPLER_BF16 if dtype == "bf16" else SAMPLER_F32, penalty_mode,
                      device)
        h = C.c_void_p()
        rc = _lib.sampler_create(C.byref(cfg), C.byref(h))
        if rc != 0:
            raise SamplerError(rc, _lib.sampler_last_error(None).decode())
        self.h = h
        self.cfg = cfg
        self.dtype = dtype
        self.device = device

    # ------------------------------------------------------------------ state
    def _check(self, rc):
        if rc != 0:
            raise SamplerError(rc, _lib.sampler_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            _lib.sampler_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, slots, params):
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        arr = pack_params(params)
        self._check(_lib.sampler_set_params(self.h, len(slots), slots.ctypes.data_as(C.c_void_p),
                                            arr.ctypes.data_as(C.c_void_p)))

    def set_history(self, slot, prompt=(), output=()):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        o = np.ascontiguousarray(output, dtype=np.int32)
        self._check(_lib.sampler_set_history(self.h, int(slot), p.ctypes.data_as(C.c_void_p), len(p),
                                             o.ctypes.data_as(C.c_void_p), len(o)))

    def append_tokens(self, slots, tokens):
        s = np.ascontiguousarray(slots, dtype=np.int32)
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        self._check(_lib.sampler_append_tokens(self.h, len(s), s.ctypes.data_as(C.c_void_p),
                                               t.ctypes.data_as(C.c_void_p)))

    def get_history(self, slot):
        L = self.cfg.max_history
        np_, no, nu = C.c_int32(), C.c_int32(), C.c_int32()
        pr, out = np.zeros(L, np.int32), np.zeros(L, np.int32)
        ids, cnt, inp = np.zeros(L, np.int32), np.zeros(L, np.int32), np.zeros(L, np.int32)
        v = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(_lib.sampler_get_history(self.h, int(slot), C.byref(np_), C.byref(no), v(pr), v(out),
                                             C.byref(nu), v(ids), v(cnt), v(inp)))
        n, m, k = np_.value, no.value, nu.value
        return dict(prompt=pr[:n].tolist(), output=out[:m].tolist(), uniq_ids=ids[:k].tolist(),
                    uniq_counts=cnt[:k].tolist(), uniq_in_prompt=inp[:k].tolist())

    def slot_flags(self, slot) -> int:
        """Bit 0 (SLOT_OVERFLOW): an append found the slot's history full and dropped the token."""
        f = C.c_int32()
        self._check(_lib.sampler_get_slot_flags(self.h, int(slot), C.byref(f)))
        return int(f.value)

    def set_step_source(self, step_dev=None):
        """step_dev: a device int64 tensor of one element (or None): later calls read the Philox step from
        it on the device (CUDA-graph replays of a decode loop advance it), ignoring their `step` argument."""
        self._step_src = step_dev  # (kept alive with the handle)
        self._check(_lib.sampler_set_step_source(self.h, _ptr(step_dev)))

    def last_launch_count(self) -> int:
        return int(_lib.sampler_last_launch_count(self.h))

    def set_timing(self, enable=True):
        """Record CUDA events around each kernel of every following call (not under graph capture)."""
        self._check(_lib.sampler_set_timing(self.h, 1 if enable else 0))

    def kernel_times_ms(self):
        """Per-kernel durations (ms, launch order) of the last call; waits for it."""
        buf = (C.c_float * 8)()
        n = C.c_int32(0)
        self._check(_lib.sampler_kernel_times(self.h, buf, 8, C.byref(n)))
        return [float(buf[i]) for i in range(n.value)]

    def record_bytes(self, B) -> int:
        return int(_lib.sampler_record_bytes(self.h, B))

    # ------------------------------------------------------------------ sampling
    def _outs(self, B, out):
        import torch
        dev = torch.device("cuda", self.device)
        if out is None:
            out = dict(tokens=torch.empty(B, dtype=torch.int32, device=dev),
                       logprobs=torch.empty(B, dtype=torch.float32, device=dev),
                       filtered_logprobs=torch.empty(B, dtype=torch.float32, device=dev),
                       status=torch.empty(B, dtype=torch.int32, device=dev))
        return out

    def sample(self, logits, step, slots=None, params=None, seeds=None, append=False, out=None, stream=None):
        """logits: [B, V] (row stride = logits.stride(0)).  params: optional device uint8 tensor of
        packed sampling_params (see pack_params) per row; None => the slot table."""
        B = logits.shape[0]
        out = self._outs(B, out)
        self._check(_lib.sampler_sample(
            self.h, _ptr(logits), logits.stride(0), B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, int(bool(append)), _ptr(out["tokens"]), _ptr(out["logprobs"]),
            _ptr(out.get("filtered_logprobs")), _ptr(out.get("status")), _stream(stream)))
        return out

    def debug_distribution(self, logits, step, slots=None, params=None, seeds=None, stream=None):
        import torch
        B = logits.shape[0]
        out = self._outs(B, None)
        q = torch.empty((B, self.cfg.vocab_size), dtype=torch.float32, device=logits.device)
        self._check(_lib.sampler_debug_distribution(
            self.h, _ptr(logits), logits.stride(0), B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, _ptr(out["tokens"]), _ptr(out["logprobs"]), _ptr(q), _stream(stream)))
        out["q"] = q
        return out

    def sample_local(self, logits_slice, records, slots=None, params=None, stream=None):
        B = logits_slice.shape[0]
        self._check(_lib.sampler_sample_local(self.h, _ptr(logits_slice), logits_slice.stride(0), B, _ptr(slots),
                                              _ptr(params), _ptr(records), _stream(stream)))

    def merge(self, gathered, world, B, step, slots=None, params=None, seeds=None, append=False, out=None,
              stream=None):
        out = self._outs(B, out)
        self._check(_lib.sampler_merge(
            self.h, _ptr(gathered), world, B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, int(bool(append)), _ptr(out["tokens"]), _ptr(out["logprobs"]),
            _ptr(out.get("filtered_logprobs")), _ptr(out.get("status")), _stream(stream)))
        return out

    # ------------------------------------------------------------------ NEXT-1 resolve rounds
    def resolve_bytes(self, B) -> int:
        return int(_lib.sampler_resolve_bytes(self.h, B))

    @staticmethod
    def resolve_max_rounds() -> int:
        return int(_lib.sampler_resolve_max_rounds())

    def resolve_round(self, logits_slice, step, rnd, gathered, world, rank, payload, out, slots=None, params=None,
                      seeds=None, append=False, active=None, stream=None):
        """One round of the sharded resolve protocol (include/sampler.h, sampler_resolve_round): ingest the
        previous round's all-gathered payloads (None at round 0), write this round's payload."""
        B = logits_slice.shape[0]
        self._check(_lib.sampler_resolve_round(
            self.h, _ptr(logits_slice), logits_slice.stride(0), B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, int(rnd), _ptr(gathered), int(world), int(rank), _ptr(payload),
            int(bool(append)), _ptr(out["tokens"]), _ptr(out["logprobs"]), _ptr(out.get("filtered_logprobs")),
            _ptr(out.get("status")), _ptr(active), _stream(stream)))

    # ------------------------------------------------------------------ NEXT-2 one-shot peer exchange
    def exchange_init(self, world, rank, timeout_ms=0):
        """Returns (64-byte IPC handle as bytes, device base address)."""
        hbuf = (C.c_uint8 * 64)()
        base = C.c_void_p()
        self._check(_lib.sampler_exchange_init(self.h, int(world), int(rank), int(timeout_ms), hbuf, C.byref(base)))
        return bytes(hbuf), int(base.value or 0)

    def exchange_open(self, handles: bytes):
        buf = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
        self._check(_lib.sampler_exchange_open(self.h, buf))

    def exchange_set_peers(self, bases):
        arr = (C.c_void_p * len(bases))(*bases)
        self._check(_lib.sampler_exchange_set_peers(self.h, arr))

    def sample_exchange(self, logits_slice, step, slots=None, params=None, seeds=None, append=False, out=None,
                        phases=3, stream=None):
        B = logits_slice.shape[0]
        out = self._outs(B, out)
        self._check(_lib.sampler_sample_exchange(
            self.h, _ptr(logits_slice), logits_slice.stride(0), B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, int(bool(append)), _ptr(out["tokens"]), _ptr(out["logprobs"]),
            _ptr(out.get("filtered_logprobs")), _ptr(out.get("status")), int(phases), _stream(stream)))
        return out

    def resolve_round_exchange(self, logits_slice, step, rnd, out, slots=None, params=None, seeds=None, append=False,
                               active=None, stream=None):
        """One resolve round through the peer exchange (no collective; after exchange_init / open)."""
        B = logits_slice.shape[0]
        self._check(_lib.sampler_resolve_round_exchange(
            self.h, _ptr(logits_slice), logits_slice.stride(0), B, _ptr(slots), _ptr(params), _ptr(seeds),
            int(step) & 0xFFFFFFFFFFFFFFFF, int(rnd), int(bool(append)), _ptr(out["tokens"]), _ptr(out["logprobs"]),
            _ptr(out.get("filtered_logprobs")), _ptr(out.get("status")), _ptr(active), _stream(stream)))


def params_to_device(params, device=0):
    """Pack per-row params into a device uint8 tensor usable as `params=` of sample()."""
    import torch
    arr = pack_params(params)
    return torch.from_numpy(arr.view(np.uint8).copy()).to(torch.device("cuda", device))

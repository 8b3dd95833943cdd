"""The paper's CPU sampling design (column-wise layout, incremental penalty buffers, AVX-512,
multi-worker) as a comparator for bench.py.

Not the product path and not the oracle: a float32 / float64-sum production-style CPU sampler
(sampler_cpu.c) that bench.py times on the host cores next to the GPU number.  Argument
marshalling only; the C library is built in-tree by `build()` (gcc, -march=x86-64-v4)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "sampler_cpu.c")
LIB = os.path.join(_HERE, "libpaper_cpu.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O3", "-march=x86-64-v4", "-fPIC", "-shared", "-o", LIB, SRC, "-lpthread", "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        _lib.pc_create.restype = C.c_void_p
        _lib.pc_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        _lib.pc_destroy.argtypes = [C.c_void_p]
        _lib.pc_set_params.argtypes = [C.c_void_p, C.c_int, C.c_float, C.c_int32, C.c_float, C.c_float, C.c_float,
                                       C.c_float, C.c_float, C.c_uint64, C.c_uint64]
        _lib.pc_set_history.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _lib.pc_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                                 C.c_int]
    return _lib


class PaperCpuSampler:
    """B requests x V vocabulary; histories up to max_output tokens of output per request."""

    def __init__(self, V: int, B: int, max_output: int = 4096, threads: int | None = None):
        lib = _load()
        self.V, self.B = V, B
        self.threads = threads or len(os.sched_getaffinity(0))
        self.h = lib.pc_create(B, V, max_output, self.threads)
        if not self.h:
            raise MemoryError("pc_create failed")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.pc_destroy(self.h)
            self.h = None

    def set_params(self, b: int, p) -> None:
        _lib.pc_set_params(self.h, b, float(p.temperature), int(p.top_k), float(p.top_p), float(p.min_p),
                           float(p.repetition_penalty), float(p.presence_penalty), float(p.frequency_penalty),
                           int(p.seed) & 0xFFFFFFFFFFFFFFFF, int(p.request_id) & 0xFFFFFFFFFFFFFFFF)

    def set_history(self, b: int, prompt, output) -> None:
        pr = np.ascontiguousarray(prompt, dtype=np.int32)
        ou = np.ascontiguousarray(output, dtype=np.int32)
        if _lib.pc_set_history(self.h, b, pr.ctypes.data, len(pr), ou.ctypes.data, len(ou)) != 0:
            raise ValueError("history longer than max_output")

    def step(self, logits: np.ndarray, step: int, append: bool = False):
        """logits: [B, ld] uint16 (bf16 bit patterns) or float32, C-contiguous.  Returns (tokens,
        logprobs)."""
        x = np.ascontiguousarray(logits)
        bf = x.dtype == np.uint16
        if not bf and x.dtype != np.float32:
            raise TypeError("logits must be uint16 (bf16 bits) or float32")
        tok = np.empty(self.B, np.int32)
        lp = np.empty(self.B, np.float32)
        _lib.pc_step(self.h, x.ctypes.data, int(bf), x.shape[1], int(step), tok.ctypes.data, lp.ctypes.data,
                     int(append))
        return tok, lp

"""B200-native last-stage LLM sampler (arXiv 2506.22033 "SiPipe" §2.1/§5.1 sampling task).

logits [B x V] (bf16/fp32, in HBM) -> penalties -> temperature -> softmax -> top-k/top-p/min-p
-> Philox-seeded categorical draw + logprobs, in hand-written sm_100a kernels behind the C ABI
of include/sampler.h.  See DESIGN.md.
"""
from .sampler import (  # noqa: F401
    Sampler, SamplingParams, SamplerError, pack_params, params_to_device, version, lib, EXPORTED,
    ROW_OK, ROW_NONFINITE, ROW_ALL_NEG_INF, ROW_UNRESOLVED, ROW_INVALID, ROW_EXCHANGE_TIMEOUT, PEN_OPENAI_CTRL, PEN_LINEAR,
)

"""CPU float64 oracle of the sampling hot path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` arm.  Shares no code with paper_2506_22033_b200/.
"""
from .philox import philox4x32_10, uniform  # noqa: F401
from .sampler_ref import (  # noqa: F401
    Params, RowResult, sample_row, sample_batch, apply_penalties, decode_logits,
    order_pi, top_k_set, top_p_set, min_p_set, draw_from,
    PEN_OPENAI_CTRL, PEN_LINEAR, ROW_OK, ROW_NONFINITE, ROW_ALL_NEG_INF,
)

"""C-ABI boundary: the library loads and exports every symbol include/sampler.h declares (CPU),
and every argument / range error is reported before any launch (GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sampler.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sampler_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2506_22033_b200.sampler import LIB_PATH, EXPORTED
    lib = ctypes.CDLL(LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(EXPORTED) == syms


def test_sass_is_sm100a_with_streaming_loads():
    """The built library contains sm_100a SASS; the streaming pass uses 16-byte read-only
    no-L1-allocate loads (LDG.E.NA.128.CONSTANT) and the hardware exp2 (MUFU.EX2)."""
    import shutil
    import subprocess
    from paper_2506_22033_b200.sampler import LIB_PATH
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([cuobjdump, "-lelf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([cuobjdump, "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "LDG.E.NA.128.CONSTANT" in sass
    assert "MUFU.EX2" in sass


def test_param_struct_layout():
    from paper_2506_22033_b200.sampler import CParams, PARAMS_DTYPE
    assert ctypes.sizeof(CParams) == 48 == PARAMS_DTYPE.itemsize
    for name, _ in CParams._fields_:
        assert getattr(CParams, name).offset == PARAMS_DTYPE.fields[name][1]


@pytest.mark.gpu
def test_error_paths_before_launch():
    import torch
    from paper_2506_22033_b200 import Sampler, SamplerError, SamplingParams
    from paper_2506_22033_b200.sampler import SAMPLER_EINVAL, SAMPLER_ERANGE, lib, CConfig
    # create errors
    h = ctypes.c_void_p()
    for cfg in (CConfig(0, 0, 0, 4, 16, 8, 2, 0, 0), CConfig(100, 0, 100, 0, 16, 8, 2, 0, 0),
                CConfig(100, 0, 100, 4, 16, 0, 2, 0, 0), CConfig(100, 0, 100, 4, 16, 8, 7, 0, 0),
                CConfig(100, 50, 60, 4, 16, 8, 2, 0, 0)):
        assert lib().sampler_create(ctypes.byref(cfg), ctypes.byref(h)) < 0
        assert not h.value
        assert lib().sampler_last_error(None)
    s = Sampler(1000, 8, max_history=16, dtype="bf16")
    bad = [SamplingParams(temperature=-1), SamplingParams(top_p=0.0), SamplingParams(top_p=1.5),
           SamplingParams(min_p=-0.1), SamplingParams(min_p=1.1), SamplingParams(repetition_penalty=0.0),
           SamplingParams(presence_penalty=float("nan"))]
    for p in bad:
        with pytest.raises(SamplerError) as e:
            s.set_params([0], [p])
        assert e.value.code == SAMPLER_EINVAL
    with pytest.raises(SamplerError) as e:
        s.set_params([8], [SamplingParams()])
    assert e.value.code == SAMPLER_ERANGE
    with pytest.raises(SamplerError) as e:
        s.set_history(0, [1] * 10, [2] * 7)  # 17 > L_max 16
    assert e.value.code == SAMPLER_ERANGE
    with pytest.raises(SamplerError) as e:
        s.set_history(0, [1000], [])
    assert e.value.code == SAMPLER_ERANGE
    with pytest.raises(SamplerError) as e:
        s.append_tokens([0], [-1])
    assert e.value.code == SAMPLER_ERANGE
    x = torch.zeros((9, 1000), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(SamplerError) as e:
        s.sample(x, 0)  # B=9 > max_batch
    assert e.value.code == SAMPLER_EINVAL
    y = torch.zeros((4, 1003), dtype=torch.bfloat16, device="cuda")[:, :1000]
    with pytest.raises(SamplerError) as e:
        s.sample(y, 0)  # ld*2 % 16 != 0
    assert e.value.code == SAMPLER_EINVAL
    # nothing was written by the failed calls
    h0 = s.get_history(0)
    assert h0["prompt"] == [] and h0["output"] == []
    # overflow through append
    s.set_history(1, [5] * 15, [])
    s.append_tokens([1], [6])
    with pytest.raises(SamplerError) as e:
        s.append_tokens([1], [7])
    assert e.value.code == SAMPLER_ERANGE
    assert s.get_history(1)["output"] == [6]


@pytest.mark.gpu
def test_in_kernel_append_overflow_sets_slot_flag():
    """An in-kernel append into a full history drops the token and sets SAMPLER_SLOT_OVERFLOW, readable
    with sampler_get_slot_flags; set_history clears it."""
    import torch
    from paper_2506_22033_b200 import Sampler
    s = Sampler(1000, 2, max_history=8, dtype="bf16")
    s.set_history(0, [1, 2, 3], [4, 5, 6, 7])   # 7 of 8
    s.set_history(1, [1], [])
    x = torch.randn((2, 1000), device="cuda").to(torch.bfloat16)
    o1 = s.sample(x, 0, append=True)
    torch.cuda.synchronize()
    assert s.slot_flags(0) == 0 and len(s.get_history(0)["output"]) == 5
    s.sample(x, 1, append=True)
    torch.cuda.synchronize()
    assert s.slot_flags(0) & 1 and len(s.get_history(0)["output"]) == 5   # dropped, flagged
    assert s.slot_flags(1) == 0 and len(s.get_history(1)["output"]) == 2
    assert int(o1["tokens"][0].item()) == s.get_history(0)["output"][-1]
    s.set_history(0, [1], [])
    assert s.slot_flags(0) == 0

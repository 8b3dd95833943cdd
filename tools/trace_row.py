"""Development timeline of the row kernel: builds a separate -DSMP_TRACE library (never the product
.so), runs one c3-shaped step and prints per-event timestamps relative to the first row start.
   python tools/trace_row.py [config] [B]
Events: producer 0 slot free / 1 copies issued; group 2 data landed / 3 A1 done / 4 pen counts in /
5 bound T / 6 A2 done / 7 record sent; decider 12 records in / 13 top-k / 14 decided."""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2506_22033_b200 import build  # noqa: E402

lib = os.path.join(ROOT, "gpurun_out", "libsampler_trace.so")
os.makedirs(os.path.dirname(lib), exist_ok=True)
build.build(force=True, out=lib, extra=["-DSMP_TRACE"])
src = open(os.path.join(ROOT, "paper_2506_22033_b200", "sampler.py")).read()
src = src.replace('LIB_PATH = os.path.join(_HERE, "libsampler_b200.so")', f'LIB_PATH = {lib!r}')
mod = types.ModuleType("sampler_trace")
sys.modules["sampler_trace"] = mod
mod.__file__ = os.path.join(ROOT, "paper_2506_22033_b200", "sampler.py")
exec(compile(src, mod.__file__, "exec"), mod.__dict__)

import ctypes as C  # noqa: E402
import torch  # noqa: E402
from workloads.synth import make_workload, device_logits  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = make_workload(cfg, B=B)
s = mod.Sampler(wl.V, wl.B, max_history=2048, max_top_k=128, dtype=wl.dtype)
s.set_params(list(range(wl.B)), wl.params)
for b in range(wl.B):
    s.set_history(b, wl.prompts[b], wl.outputs[b])
x = device_logits(wl)
for i in range(3):
    s.sample(x, i)
torch.cuda.synchronize()
nsm = torch.cuda.get_device_properties(0).multi_processor_count
n = 16 * 64 * 2 * nsm
buf = (C.c_uint64 * n)()
rc = mod._lib.sampler_debug_trace(s.h, buf, n)
assert rc == 0, rc
t = np.frombuffer(buf, dtype=np.uint64).reshape(2 * nsm, 64, 16).astype(np.int64)
tt = t.copy(); tt[:, :, 8:11] = 0
nz = tt[tt > 0]
t0 = nz.min()
rel = np.where(tt > 0, tt - t0, -1)
names = {0: "p:buf-free", 1: "p:issued", 2: "s:landed", 3: "s:passed", 4: "f:start", 5: "f:bound-xchg",
         7: "f:sent", 12: "d:recs-in", 13: "d:topk", 14: "d:decided"}
print("end of step (last stamp): %.2f us" % ((nz.max() - t0) / 1e3))
for ev, nm in names.items():
    v = rel[:, :, ev]
    v = v[v >= 0]
    if len(v):
        print(f"{nm:12s} n={len(v):5d} min={v.min()/1e3:8.2f} p50={np.median(v)/1e3:8.2f} max={v.max()/1e3:8.2f} us")
v = t[:, :, 8][t[:, :, 2] > 0]
print("candidates per chunk: mean %.1f max %d" % (v.mean(), v.max()))
print("tkey/rkey row0 CTA0..3:", [(hex(int(t[c, 0, 9])), hex(int(t[c, 0, 10]))) for c in range(4)])
# per-row phase durations (CTA 0's rows)
print("CTA 0 rows (us): it: landed passed | fin-start bound-xchg sent | dec: in topk decided")
for it in range(min(12, 64)):
    r = rel[0, it]
    if r[2] < 0:
        break
    f = lambda e: ("%7.2f" % (r[e] / 1e3)) if r[e] >= 0 else "      -"
    print(it, " ".join(f(e) for e in (2, 3)), "|", " ".join(f(e) for e in (4, 5, 7)), "|", " ".join(f(e) for e in (12, 13, 14)))

#!/bin/bash
# Development: per-phase globaltimer marks of exact_kernel (rows 0-2) for one config.  Builds an
# EXACT_PROF copy of the library in place (on the GPU box's scratch copy only).  Output gpurun_out/$1/.
TAG=${1:-marks}; CFG=${2:-c2}
O=gpurun_out/$TAG; mkdir -p $O
python -c "from paper_2506_22033_b200.build import build; build(force=True, extra=['-DEXACT_PROF'])"
python - "$CFG" > $O/marks_$CFG.txt 2>&1 <<'PY'
import sys, torch
from tests._helpers import make_sampler
from workloads.synth import device_logits, make_workload
wl = make_workload(sys.argv[1])
s = make_sampler(wl); x = device_logits(wl)
for i in range(3):
    s.sample(x, i); torch.cuda.synchronize()
    print("---", flush=True)
PY
python tools/exact_marks.py $O/marks_$CFG.txt

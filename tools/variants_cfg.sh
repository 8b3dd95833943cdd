#!/bin/bash
# A/B of the .variants/*.so builds on one config: bash tools/variants_cfg.sh CFG STEPS
CFG=${1:-c2}; STEPS=${2:-200}
for r in 1 2; do for f in .variants/*.so; do
  cp $f paper_2506_22033_b200/libsampler_b200.so
  timeout 300 python bench.py --config $CFG --steps $STEPS --warmup 10 --no-cpu-baseline --e2e-steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$f', round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['roofline']['kernel_times_us'].items()})"
done; done
cp .variants/base.so paper_2506_22033_b200/libsampler_b200.so

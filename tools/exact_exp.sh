#!/bin/bash
# Development: exact_kernel time (c2 bench) for EXACT_EXP variants (timing only).
O=gpurun_out/${1:-exps}; mkdir -p $O; CFG=${2:-c2}
for i in ${EXPS:-0 1 2 3}; do
  python -c "from paper_2506_22033_b200.build import build; build(force=True, extra=['-DEXACT_EXP=$i'])"
  timeout 300 python bench.py --config $CFG --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $O/e$i.json 2> $O/e$i.err
  python -c "import json; d=json.load(open('$O/e$i.json')); print('exp $i', round(d['roofline']['kernel_times_us'].get('exact_kernel', 0), 1))"
done

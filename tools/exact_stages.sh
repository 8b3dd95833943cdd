#!/bin/bash
# Development: exact_kernel time (c2 bench) when the kernel leaves after stage i (EXACT_STOP builds;
# results invalid, timing only).  Output gpurun_out/$1/.
O=gpurun_out/${1:-stages}; mkdir -p $O; CFG=${2:-c2}
for i in ${STAGES:-2 3 4 12 13 14 99}; do
  python -c "from paper_2506_22033_b200.build import build; build(force=True, extra=['-DEXACT_STOP=$i'])"
  timeout 300 python bench.py --config $CFG --steps 100 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $O/s$i.json 2> $O/s$i.err
  python -c "import json; d=json.load(open('$O/s$i.json')); print('stop $i', round(d['roofline']['kernel_times_us'].get('exact_kernel', 0), 1))"
done

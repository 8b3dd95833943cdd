#!/bin/bash
# NEXT-4: c3 step time vs history length per row (bench.py --hist).  Output gpurun_out/$1/.
O=gpurun_out/${1:-hist}; mkdir -p $O
for n in ${HISTS:-512 4096 32768 131072}; do
  timeout 900 python bench.py --config ${CFG:-c3} --hist $n --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 3 > $O/h$n.json 2> $O/h$n.err
  python -c "import json; d=json.load(open('$O/h$n.json')); print('hist $n', 'ms/step', round(d['ms_per_step'],4), 'kernels', {k: round(v,1) for k,v in d['roofline']['kernel_times_us'].items()}, d['config']['history'][:40])" || tail -3 $O/h$n.err
done

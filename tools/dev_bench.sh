#!/bin/bash
# Development: c2 / c4 bench lines (exact kernel times).  Output gpurun_out/$1/.
O=gpurun_out/${1:-db}; mkdir -p $O
for c in ${2:-c2 c4}; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 3 > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in ${2:-c2 c4}; do python -c "import json,sys; d=json.load(open('$O/bench_$c.json')); print('$c', round(d['ms_per_step']*1000,1), 'us', {k: round(v,1) for k,v in d['roofline']['kernel_times_us'].items()})"; done

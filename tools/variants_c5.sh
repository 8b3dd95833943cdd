#!/bin/bash
# A/B of the .variants/*.so builds on c5 batch sizes: bash tools/variants_c5.sh "1 8 32"
for r in 1 2; do for B in ${1:-1 32}; do for f in .variants/*.so; do
  cp $f paper_2506_22033_b200/libsampler_b200.so
  timeout 300 python bench.py --config c5 --batch $B --steps 1000 --warmup 20 --no-cpu-baseline --e2e-steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 B=$B', '$f', round(d['ms_per_step']*1e3,2), {k: round(v,1) for k,v in d['roofline']['kernel_times_us'].items()})"
done; done; done
cp .variants/base.so paper_2506_22033_b200/libsampler_b200.so

#!/bin/bash
# Every BASELINE config once (short runs, no CPU baseline): one JSON line each.  Output gpurun_out/$TAG/.
TAG=${TAG:-cfg}
O=gpurun_out/$TAG
mkdir -p $O
for c in c1 c2 c3 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?" >> $O/rc.txt
done
for b in 1 2 4 8 16 32; do
  timeout 300 python bench.py --config c5 --batch $b --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 5 > $O/bench_c5_b$b.json 2> $O/bench_c5_b$b.err
  echo "c5 b$b rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['config']['workload'], d['config']['B'], 'ms/step=%.4f'%d['ms_per_step'], 'rows/s=%.3g'%d['value'], 'kern=', r.get('kernel_times_us'), 'frac=%.3f'%r['frac'])" 2>/dev/null || (echo "$f FAILED"; tail -5 ${f%.json}.err); done

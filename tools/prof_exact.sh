#!/bin/bash
# ncu --set full of one exact_kernel launch (c2 bench configuration).  Output gpurun_out/$1/.
TAG=${1:-pex}; CFG=${2:-c2}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exact_kernel -s 2 -c 1 \
  -o $O/full python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3 > $O/ncu_full.log 2>&1
tail -3 $O/ncu_full.log

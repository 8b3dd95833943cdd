#!/bin/bash
# ncu --set full of one row_kernel launch in the c3 bench configuration.  Output gpurun_out/$1/.
TAG=${1:-prof}; CFG=${2:-c3}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:row_kernel -s 6 -c 1 \
  -o $O/full python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 3 > $O/ncu_full.log 2>&1
tail -3 $O/ncu_full.log

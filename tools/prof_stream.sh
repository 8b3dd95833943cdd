#!/bin/bash
# ncu --set full of one stream_kernel + one select_rows_kernel launch of the c3 bench (no graphs).
TAG=${TAG:-p}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|select_rows" -s 6 -c 2 \
  -o $O/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_full.log 2>&1
tail -3 $O/ncu_full.log

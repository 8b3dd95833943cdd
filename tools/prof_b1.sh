#!/bin/bash
# ncu source-level profile of phase B at B=1 (latency chain of one row).
TAG=${TAG:-pb1}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"select_rows" -s 5 -c 1 \
  -o $O/full python bench.py --config c5 --batch 1 --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu.log 2>&1
tail -2 $O/ncu.log

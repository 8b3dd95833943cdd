#!/bin/bash
# ncu of the exact kernel on c2 (top-p-only rows)
TAG=${TAG:-pex}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exact_kernel" -s 2 -c 1 \
  -o $O/full python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu.log 2>&1
tail -2 $O/ncu.log

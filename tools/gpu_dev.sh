#!/bin/bash
# Development GPU check: GPU tests (first failure stops), a short c3 bench.  Output under gpurun_out/$TAG/.
TAG=${1:-dev}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/ -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
tail -30 $O/pytest_gpu.log; cat $O/bench.json; tail -5 $O/bench.err

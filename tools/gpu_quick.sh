#!/bin/bash
# Quick GPU check: parity tests, a short bench, the launch list, the phase trace.  Output under gpurun_out/$TAG/.
TAG=${TAG:-q}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/ -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_bench.log 2>&1
timeout 120 python tools/trace.py c3 > $O/trace.txt 2>&1
tail -3 $O/pytest_gpu.log; cat $O/bench.json; tail -3 $O/bench.err
python tools/launches.py $O/launches.csv 2>/dev/null | tail -12
cat $O/trace.txt

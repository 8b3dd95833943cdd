#!/bin/bash
# One GPU session: parity tests, bench (both arms), ncu launch list + full capture of the two
# phase kernels.  Output under gpurun_out/$TAG/.
TAG=${TAG:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,driver_version --format=csv >> $O/smi.txt 2>&1; nproc >> $O/smi.txt; lscpu | head -20 >> $O/smi.txt
timeout 600 python -m pytest tests/ -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv 2>&1 &
SMI=$!
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
kill $SMI 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|select_rows" -s 6 -c 2 \
  -o $O/full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_full.log 2>&1
tail -2 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/bench.json; tail -3 $O/bench.err; cat $O/bench_ref.json; tail -3 $O/ncu_full.log

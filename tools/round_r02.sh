#!/bin/bash
# Round-2 evidence: every config's bench line, the c3 bench with the CPU baseline, the reference arm,
# clocks, the ncu launch list (c3 and c2) and ncu --set full of each kernel.  Output gpurun_out/$1/.
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,driver_version --format=csv > $O/smi.txt 2>&1; nproc >> $O/smi.txt; lscpu | head -20 >> $O/smi.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv 2>&1 &
SMI=$!
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
kill $SMI 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in c1 c2 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
done
for b in 1 2 4 8 16 32; do
  timeout 300 python bench.py --config c5 --batch $b --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 5 > $O/bench_c5_b$b.json 2> $O/bench_c5_b$b.err
done
# vocab-sharded step at world 1 (one-shot peer exchange vs NCCL all-gather; c2 with the resolve rounds)
for ex in p2p nccl; do
  timeout 300 python bench.py --shard vocab --exchange $ex --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 5 > $O/bench_c3_vocab1_$ex.json 2> $O/bench_c3_vocab1_$ex.err
done
timeout 300 python bench.py --shard vocab --config c2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 3 > $O/bench_c2_vocab1_p2p.json 2> $O/bench_c2_vocab1_p2p.err
# parity statistics (unsharded >= 1e5 rows; vocab-sharded G = 4)
[ -n "$PARITY" ] && timeout 1500 python tools/parity_stats.py --rows 100000 --out $O/parity.json > $O/parity.log 2>&1
[ -n "$PARITY" ] && timeout 900 python tools/parity_stats.py --rows 40000 --sharded 4 --out $O/parity_sharded4.json > $O/parity_sharded4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2.csv \
  python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|select_rows" -s 6 -c 2 \
  -o $O/full_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exact_kernel" -s 2 -c 1 \
  -o $O/full_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph --e2e-steps 0 > $O/ncu_full_c2.log 2>&1
ls $O

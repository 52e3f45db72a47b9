#!/bin/bash
# Round-2 measurement batch (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"
done
timeout 600 python bench.py --hero --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_hero.log 2>&1; echo "bench hero rc=$?"
timeout 900 python bench.py --literal --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_literal.log 2>&1; echo "bench literal rc=$?"
L="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 300 $L > gpurun_out/launch_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg4.csv $L > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
for c in 4 2 3; do
  P="python bench.py --config $c --outputs 1024 --steps 1 --warmup 0 --no-cpu --no-e2e"
  timeout 300 $P > gpurun_out/prof_plain_$c.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:lofp_units_kernel -s 1 -c 1 -o gpurun_out/r2_units_cfg$c $P > gpurun_out/ncu_full_$c.log 2>&1; echo "ncu cfg$c rc=$?"
done

#!/bin/bash
# Round-2 measurement batch (run under gpurun from the repo root).  TAG names the outputs.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_cfg4.log 2>&1; echo "bench cfg4 rc=$?"
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"
done
timeout 600 python bench.py --hero --steps 3 --warmup 3 --no-e2e > gpurun_out/${TAG}_bench_hero.log 2>&1; echo "bench hero rc=$?"
timeout 900 python bench.py --literal --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_literal.log 2>&1; echo "bench literal rc=$?"
timeout 600 python bench.py --contract --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_contract_cfg3.log 2>&1; echo "bench contract rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference_cfg4.log 2>&1; echo "reference rc=$?"
L="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 300 $L > gpurun_out/launch_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg4.csv $L > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
for c in 4 2 3; do
  P="python bench.py --config $c --steps 1 --warmup 0 --no-cpu --no-e2e"
  timeout 300 $P > gpurun_out/prof_plain_$c.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:lofp_units_kernel -s 1 -c 1 -o gpurun_out/${TAG}_units_cfg$c $P > gpurun_out/ncu_full_$c.log 2>&1; echo "ncu cfg$c rc=$?"
done
P="python bench.py --contract --steps 1 --warmup 0 --no-e2e"
timeout 300 $P > gpurun_out/prof_plain_contract.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lofp_contract_warp -s 1 -c 1 -o gpurun_out/${TAG}_contract_warp_cfg3 $P > gpurun_out/ncu_full_contract.log 2>&1; echo "ncu contract rc=$?"
timeout 300 python bench.py --nonlocal --outputs 256 --steps 3 --warmup 2 --no-cpu > gpurun_out/${TAG}_bench_nonlocal.log 2>&1; echo "nonlocal rc=$?"
timeout 300 python bench.py --gates --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_gates.log 2>&1; echo "gates rc=$?"
timeout 300 python bench.py --distribution --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_distribution.log 2>&1; echo "distribution rc=$?"
timeout 600 python scripts/paper_scaling.py gpurun_out/${TAG}_paper_scaling.json > gpurun_out/${TAG}_paper_scaling.log 2>&1; echo "paper scaling rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"

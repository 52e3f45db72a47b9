#!/bin/bash
# ncu --set full of lofp_units_kernel on full conditioned batches (run under gpurun)
set -u
mkdir -p gpurun_out
TAG=${TAG:-v2}
for c in ${CFGS:-2 3 4}; do
  P="python bench.py --config $c --steps 1 --warmup 0 --no-cpu --no-e2e"
  timeout 300 $P > gpurun_out/prof_plain_$c.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:lofp_units_kernel -s 1 -c 1 -o gpurun_out/r2_${TAG}_cfg$c $P > gpurun_out/ncu_${TAG}_$c.log 2>&1; echo "ncu cfg$c rc=$?"
done

#!/bin/bash
# quick correctness + three-config bench (run under gpurun)
set -u
mkdir -p gpurun_out
NRAND=30 NCOND=256 timeout 300 python scripts/gpu_quick.py > gpurun_out/quick.log 2>&1; echo "quick rc=$? $(tail -1 gpurun_out/quick.log)"
for c in 4 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg$c.log 2>&1
  echo "cfg$c rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_cfg$c.log').read().strip().splitlines()[-1]); print('%.3e paths/s frac %.3f units %d' % (d['value'], d['roofline']['frac'], d['stats']['units']))" 2>&1 | tail -1)"
done

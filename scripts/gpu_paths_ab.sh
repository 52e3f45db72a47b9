#!/bin/bash
# Path-sum A/B under gpurun: bench lines of configs[4], [2], [3] (device value and FP64 fraction),
# the P:318 density single outputs, then the path-engine GPU tests.
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab}
for c in 4 2 3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_cfg$c.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/${TAG}_cfg$c.log') if x.startswith('{')][-1]; d=json.loads(l); print('cfg$c', '%.4e' % d['value'], 'frac %.4f' % d['roofline']['frac'], 'sm_mhz', d['clocks']['sm_mhz'])"
done
timeout 300 python scripts/density_stats.py 2>&1 | grep 'upb=2'
if [ "${TESTS:-1}" = 1 ]; then timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2; fi

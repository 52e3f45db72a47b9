#!/bin/bash
# A/B of the contraction's lanes per output on configs[3] literal (bench --contract)
for g in 32 8 16; do
  LOFP_CONTRACT_GROUP=$g timeout 300 python bench.py --contract --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/cg_$g.log 2>&1
  echo "G=$g rc=$? $(tail -1 gpurun_out/cg_$g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>/dev/null)"
done

#!/bin/bash
# A/B of liblofp variants on the contraction bench (configs[3] literal); args: variant names ("" = liblofp.so)
for rep in 1 2; do
  for v in "$@"; do
    lib=paper_2510_26408_b200/liblofp.so; [ "$v" != base ] && lib=paper_2510_26408_b200/liblofp_$v.so
    LOFP_LIB=$PWD/$lib timeout 300 python bench.py --contract --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cab_$v.log 2>&1
    echo "$v rc=$? $(tail -1 gpurun_out/cab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>/dev/null)"
  done
done

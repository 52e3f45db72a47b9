#!/bin/bash
# Contraction iteration under gpurun: contraction tests (release + debug build), bench, ncu of the warp kernel.
set -u
mkdir -p gpurun_out
TAG=${TAG:-c}
timeout 600 python -m pytest tests/test_gpu_contract.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
LOFP_LIB=$PWD/paper_2510_26408_b200/liblofp_debug.so timeout 600 python -m pytest tests/test_gpu_contract.py -x -q > gpurun_out/${TAG}_tests_dbg.log 2>&1; echo "dbg rc=$?"; tail -1 gpurun_out/${TAG}_tests_dbg.log
for rep in 1 2; do
timeout 300 python bench.py --contract --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-160
done
timeout 300 python bench.py --distribution --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_dist.log 2>&1; tail -1 gpurun_out/${TAG}_dist.log | cut -c1-160
if [ "${NCU:-1}" = 1 ]; then
P="python bench.py --contract --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lofp_contract_warp -s 1 -c 1 -o gpurun_out/${TAG}_warp $P > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
fi

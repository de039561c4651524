#!/bin/bash
# A/B of the fused-pass layouts: 2 vs 4 columns per lane (IBM_WF_CPL), parity first.
TAG=${1:-cpl}
mkdir -p gpurun_out
IBM_WF_CPL=4 python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}_cpl4.log 2>&1
tail -3 gpurun_out/pytest_${TAG}_cpl4.log
for CPL in 2 4; do
  for L in 128 256; do
    echo "cpl=$CPL L=$L $(IBM_WF_CPL=$CPL IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done | tee gpurun_out/mb_${TAG}.txt
IBM_WF_CPL=4 IBM_WF_ROWS=128 ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf4_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf4_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf4_${TAG}.log

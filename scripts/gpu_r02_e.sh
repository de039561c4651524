#!/bin/bash
# k_sor_wf occupancy variants (2 stages, refill after step 0) + the resident mid-grid solve
TAG=${1:-r02e}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
grep -E "^(FAILED|E )" gpurun_out/pytest_${TAG}.log | head -20
timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}.json > gpurun_out/mid_tb_${TAG}.log 2>&1; tail -8 gpurun_out/mid_tb_${TAG}.log
for mb in 8 10 12; do
  IBM_NVCC_DEFS="-DWF_MINB=$mb" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 128 256; do
    echo "minb=$mb L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done | tee gpurun_out/mb_${TAG}.txt
python paper_2402_17337_b200/build.py --force > /dev/null 2>&1

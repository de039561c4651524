#!/bin/bash
# NS (column pairs per lane) experiment for the fused pass
mkdir -p gpurun_out
for NS in 1 2; do
  IBM_NVCC_DEFS="-DWF_NS=$NS" python paper_2402_17337_b200/build.py --force > gpurun_out/build_ns$NS.log 2>&1
  for L in 64 128; do
    echo "ns=$NS rows=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 2 2>&1 | tail -1)" | tee -a gpurun_out/ns.txt
  done
  python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider 2>&1 | tail -1
done

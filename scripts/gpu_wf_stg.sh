#!/bin/bash
# stages-per-warp experiment for the fused pass
mkdir -p gpurun_out
for S in 2 3; do
  IBM_NVCC_DEFS="-DWF_NSTG=$S" python paper_2402_17337_b200/build.py --force > gpurun_out/build_stg$S.log 2>&1
  for f in 2 3; do
    echo "stg=$S fuse=$f $(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1)" | tee -a gpurun_out/stg.txt
  done
done

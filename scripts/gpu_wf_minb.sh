#!/bin/bash
# register budget experiment: resident CTAs per SM 4 / 3 / 2 for the fused pass
mkdir -p gpurun_out
for B in 4 3 2; do
  IBM_NVCC_DEFS="-DWF_MINB=$B" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 64 128; do
    for f in 2 3; do
      echo "minb=$B fuse=$f rows=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1)" | tee -a gpurun_out/minb.txt
    done
  done
done

#!/bin/bash
# fused-pass build variants: stages per warp (half windows) and column pairs per lane
TAG=${1:-r02m}
mkdir -p gpurun_out
for defs in "-DWF_NSTG=4" "-DWF_NSTG=3" "-DWF_NSTG=6" "-DWF_NS=2 -DWF_NSTG=3"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > gpurun_out/build_${TAG}.log 2>&1
  r=$(grep -A2 "k_sor_wfILi3ELi0" gpurun_out/build_${TAG}.log | grep -o "Used [0-9]* registers")
  for L in 128 256; do
    echo "defs=[$defs] $r L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done
python paper_2402_17337_b200/build.py --force > /dev/null 2>&1

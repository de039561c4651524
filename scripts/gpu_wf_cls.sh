#!/bin/bash
# edge-chunk ownership classes vs code size (cold micro-benchmark, m = 3, L = 128)
mkdir -p gpurun_out
for defs in "-DWF_OWNCLS=0" "" "-DWF_OWNCLS=0 -DWF_ONEMODE2=1" "-DWF_OWNCLS=0 -DWF_NSTG=3"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > gpurun_out/build.log 2>&1
  r=$(grep -A2 "k_sor_wfILi3ELi0" gpurun_out/build.log | grep -o "Used [0-9]* registers")
  for f in 3; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] $r fuse=$f cold $m"
  done
done

#!/bin/bash
# cold micro-benchmark of build variants: gpu_wf_defs.sh "DEFS1" "DEFS2" ...  (FUSES env: fused depths)
mkdir -p gpurun_out
for defs in "$@"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
  r=$(grep -A2 "k_sor_wfILi3ELi0" gpurun_out/build.log | grep -o "Used [0-9]* registers")
  for f in ${FUSES:-3}; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] $r fuse=$f cold $m"
  done
done

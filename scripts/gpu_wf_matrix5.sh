#!/bin/bash
# one warp per CTA: resident-warp and stage-count variants of the fused pass (cold micro-benchmark)
mkdir -p gpurun_out
for defs in "-DWF_NW=1 -DWF_MINB=8" "-DWF_NW=1 -DWF_MINB=12 -DWF_NSTG=2" "-DWF_NW=1 -DWF_MINB=8 -DWF_NSTG=2"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force 2>&1 | grep -A1 "k_sor_wfILi3ELi0" | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
  for f in 3 2 4; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] fuse=$f cold $m"
  done
done

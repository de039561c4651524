#!/bin/bash
# occupancy experiments for the m = 3 fused pass (cold micro-benchmark)
mkdir -p gpurun_out
for defs in "" "-DWF_NW=3 -DWF_MINB=3" "-DWF_NSTG=2 -DWF_MINB=3" "-DWF_NW=2 -DWF_MINB=4"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for f in 3 2; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] fuse=$f cold $m"
  done
done

#!/bin/bash
# cost of the residual in the fused pass: exact u64 max vs high-word max vs none (cold micro-benchmark)
mkdir -p gpurun_out
for defs in "" "-DWF_EXP_HI" "-DWF_EXP_NORES"; do
  IBM_NVCC_DEFS="-DWF_NW=1 -DWF_MINB=8 -DWF_NSTG=2 $defs" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for f in 3 4; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] fuse=$f cold $m"
  done
done

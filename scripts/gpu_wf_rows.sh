#!/bin/bash
# segment length L (IBM_WF_ROWS) of the fused pass, default build (cold micro-benchmark)
mkdir -p gpurun_out
python paper_2402_17337_b200/build.py --force 2>&1 | grep -A2 "k_sor_wfILi3ELi0" | grep -o "Used [0-9]* registers"
for f in 3 2; do
  for L in 64 128 192 256 512; do
    m=$(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "fuse=$f L=$L cold $m"
  done
done

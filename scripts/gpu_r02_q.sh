#!/bin/bash
# warps per SM of the fused pass now that it needs 194 registers (168 without spills at 10-12)
TAG=${1:-r02q}
mkdir -p gpurun_out
for mb in 8 10 12; do
  IBM_NVCC_DEFS="-DWF_MINB=$mb" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 128 256; do
    echo "minb=$mb L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done
python paper_2402_17337_b200/build.py --force > /dev/null 2>&1

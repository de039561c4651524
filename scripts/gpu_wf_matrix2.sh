#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider 2>&1 | tail -1
for cfg in "3 2 2" "3 3 2" "3 3 3" "3 2 3"; do
  set -- $cfg; B=$1; S=$2; F=$3
  IBM_NVCC_DEFS="-DWF_MINB=$B -DWF_NSTG=$S" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 64 128; do
  m=$(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $F 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
  echo "minb=$B stg=$S fuse=$F rows=$L cold $m"
  done
done

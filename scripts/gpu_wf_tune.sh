#!/bin/bash
# micro-benchmark of the fused Poisson pass over fuse depth x segment length
TAG=${1:-t}
mkdir -p gpurun_out
for f in ${FUSES:-2 3}; do
  for L in ${ROWS:-0 256 128}; do
    if [ "$L" != "0" ]; then export IBM_WF_ROWS=$L; else unset IBM_WF_ROWS; fi
    echo "fuse=$f rows=$L $(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1)" | tee -a gpurun_out/tune_${TAG}.txt
  done
done

#!/bin/bash
# fused Poisson pass: parity tests, then the micro-benchmark for every fuse depth
TAG=${1:-wf}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_wf_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_wf_${TAG}.log
for f in 1 2 3 4; do
  timeout 300 python scripts/microbench_sor.py 8192 1 300 $f 2>&1 | tail -1 | tee -a gpurun_out/micro_wf_${TAG}.json
done

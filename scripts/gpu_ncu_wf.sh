#!/bin/bash
# full capture of one fused Poisson pass (sor_fuse=${2:-2}) deep into the micro-benchmark
TAG=${1:-wf}
F=${2:-2}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_${TAG} -f python scripts/microbench_sor.py 8192 1 120 $F > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_wf_${TAG}.log

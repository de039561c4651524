#!/bin/bash
TAG=${1:-s}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_sor -s 14 -c 2 \
    -o gpurun_out/prof_sor_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 20 --maxit-uv 10 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_sor_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_sor_${TAG}.log

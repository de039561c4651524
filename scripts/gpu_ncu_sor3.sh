#!/bin/bash
# full capture of a Poisson SOR launch late in the second step (~iteration 9000)
TAG=${1:-s}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_sor -s 19050 -c 1 \
    -o gpurun_out/prof_sorlate_${TAG} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_sorlate_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_sorlate_${TAG}.log

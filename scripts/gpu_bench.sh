#!/bin/bash
# One GPU session: tests, bench, ncu launch list and a full capture of the top kernels.
# Usage (from the repo root, under gpurun): bash scripts/gpu_bench.sh [tag]
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
grep -E "MemTotal|MemAvailable" /proc/meminfo >> gpurun_out/gpu_${TAG}.txt; nproc >> gpurun_out/gpu_${TAG}.txt
python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 0 --maxit-p 100 --maxit-uv 20 --no-e2e --no-cpu-baseline --no-clocks > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sor<0>' -s 10 -c 2 \
    -o gpurun_out/prof_sor_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 30 --maxit-uv 10 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_sor_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_pred|k_prhs|k_correct|k_sor<1>' -c 8 \
    -o gpurun_out/prof_other_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_other_${TAG}.log 2>&1
ls -la gpurun_out

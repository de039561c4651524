#!/bin/bash
# Reports: Table-1/2-layout performance report (oracle_seq / oracle_omp / GPU, M1), the
# input-scaling sweep (BJ configs[3]) and the per-step kernels' ncu counters.
# Usage (under gpurun): bash scripts/gpu_reports.sh TAG
TAG=${1:-rep}
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python scripts/perf_report.py --level 1 --maxit-p 200 --out gpurun_out/perf_report_${TAG} > gpurun_out/perf_${TAG}.log 2>&1; tail -14 gpurun_out/perf_${TAG}.log
timeout 1200 python scripts/sweep_sizes.py --out gpurun_out/sweep_${TAG}.json > gpurun_out/sweep_${TAG}.log 2>&1; cut -c1-250 gpurun_out/sweep_${TAG}.log
ncu --set full --clock-control none --import-source on -k regex:'k_pred|k_prhs|k_correct|k_outlet|k_pext' -c 8 \
    -o gpurun_out/prof_step_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_step_${TAG}.log 2>&1

#!/bin/bash
# Round-2 profiling session: cold micro-benchmark of the fused pass at L=128/256,
# full ncu captures (source view) of k_sor_wf at both, DRAM counters of the per-step kernels.
TAG=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
for L in 128 256; do
  echo "L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1)" >> gpurun_out/mb_${TAG}.txt
done
for L in 128 256; do
  IBM_WF_ROWS=$L ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf${L}_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf${L}_${TAG}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:'k_pred|k_prhs|k_correct|k_outlet|k_forces' -c 8 \
    -o gpurun_out/prof_other_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_other_${TAG}.log 2>&1
ls -la gpurun_out | grep ${TAG}

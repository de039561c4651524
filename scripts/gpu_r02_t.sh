#!/bin/bash
# Profile HEAD: cold micro-benchmark of the fused pass, full ncu of k_sor_wf (source view),
# per-step kernels' DRAM counters, fp64/shuffle latency probe.
TAG=${1:-r02t}
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dp_latency scripts/probes/dp_latency.cu && /tmp/dp_latency > gpurun_out/dp_latency_${TAG}.txt 2>&1
cat gpurun_out/dp_latency_${TAG}.txt
timeout 300 python scripts/microbench_sor.py 8192 1 200 3 > gpurun_out/mb_${TAG}.txt 2>&1; tail -1 gpurun_out/mb_${TAG}.txt
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_wf_${TAG}.log
ncu --set full --clock-control none --import-source on -k regex:'k_pred|k_prhs|k_correct|k_outlet|k_forces|k_classify|k_pflags|k_pext' -c 12 \
    -o gpurun_out/prof_other_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_other_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_other_${TAG}.log
ls -la gpurun_out | grep ${TAG}

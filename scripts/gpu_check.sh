#!/bin/bash
# GPU check after a kernel change: parity tests, bench (JSON line), one full ncu
# capture of the fused Poisson pass (source view), the fp64 latency probe.
# Usage (repo root, under gpurun): bash scripts/gpu_check.sh TAG [FUSE]
TAG=${1:-chk}
F=${2:-3}
mkdir -p gpurun_out
bash scripts/gpu_quick.sh ${TAG}
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_${TAG} -f python scripts/microbench_sor.py 8192 1 120 $F > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_wf_${TAG}.log
python scripts/microbench_sor.py 8192 1 120 $F 2>&1 | tail -3
[ -x scripts/probes/dp_latency ] && scripts/probes/dp_latency > gpurun_out/dp_latency.txt 2>&1; cat gpurun_out/dp_latency.txt

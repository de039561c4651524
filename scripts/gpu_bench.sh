#!/bin/bash
# One GPU session: smoke, bench (JSON line), ncu launch list of the bench command
# and full captures of the Poisson SOR pass and the other kernels.
# Usage (from the repo root, under gpurun): bash scripts/gpu_bench.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
nproc >> gpurun_out/gpu_${TAG}.txt
python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_${TAG}.json
# launch list (cold-cache, serialised): the bench command with a short Poisson cap
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 0 --maxit-p 200 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > /dev/null 2>&1
# full captures: the fused Poisson pass (k_sor_wf, 3 iterations per launch) ~120 iterations into the
# first step, the one-iteration pass (--sor-fuse 1) likewise, and the other kernels
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 -o gpurun_out/prof_wf_${TAG} -f \
    python bench.py --steps 1 --warmup 0 --maxit-p 220 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_sor<.int.0' -s 40 -c 1 -o gpurun_out/prof_sor_${TAG} -f \
    python bench.py --steps 1 --warmup 0 --maxit-p 220 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 --sor-fuse 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_pred|k_prhs|k_correct|k_outlet|k_pext|k_forces' -c 12 \
    -o gpurun_out/prof_other_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_sor -s 2 -c 1 -o gpurun_out/prof_uvsor_${TAG} -f \
    python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 10 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > /dev/null 2>&1
ls gpurun_out | grep ${TAG}

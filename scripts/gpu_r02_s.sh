#!/bin/bash
# HEAD check after the session restart: GPU parity suite, smoke, full bench line (with cpu_baseline)
TAG=${1:-r02s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_${TAG}.log
python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err

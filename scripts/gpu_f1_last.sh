#!/bin/bash
bash scripts/gpu_longruns.sh foil 3 40
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_check.json 2>&1; tail -c 600 gpurun_out/bench_check.json

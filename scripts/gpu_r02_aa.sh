#!/bin/bash
# device-initiated halo (peer stores) in the decomposed fused pass: full GPU suite + micro-benchmark
TAG=${1:-r02aa}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
echo "single slab $(timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['200']['ms_per_it'])")"

#!/bin/bash
# cold micro-benchmark first, then parity tests, then the bench
TAG=${1:-p}
mkdir -p gpurun_out
python scripts/microbench_sor.py 8192 1 300 > gpurun_out/micro_${TAG}.json 2>&1; cat gpurun_out/micro_${TAG}.json | tail -1
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -1 gpurun_out/pytest_${TAG}.log
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g clocks %s' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))"

#!/bin/bash
# parity tests + bench (no ncu)
TAG=${1:-q}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -5 gpurun_out/pytest_${TAG}.log
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
cat gpurun_out/bench_${TAG}.json | python -c "import json,sys; d=json.load(sys.stdin); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value']))"
tail -3 gpurun_out/bench_${TAG}.err

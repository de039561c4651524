#!/bin/bash
TAG=${1:-r02l}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
grep -E "^(FAILED|E )" gpurun_out/pytest_${TAG}.log | head -20
for L in 128 256; do
  echo "L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
done
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g clocks %s' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))"

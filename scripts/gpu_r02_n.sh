#!/bin/bash
# residual accumulation variants (WF_RES2 = 1: two accumulators, no sign-clear LOP3) + bench
TAG=${1:-r02n}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -1 gpurun_out/pytest_${TAG}.log
for defs in "-DWF_RES2=0" "-DWF_RES2=1"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 128 256; do
    echo "defs=[$defs] L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done
python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g clocks %s' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))"

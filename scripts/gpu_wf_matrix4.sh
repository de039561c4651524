#!/bin/bash
# warps per CTA for the m = 3 fused pass (cold micro-benchmark), then the default build's bench
mkdir -p gpurun_out
for defs in "-DWF_NW=1 -DWF_MINB=8" "-DWF_NW=2 -DWF_MINB=4" ""; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for f in 3; do
    m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "defs=[$defs] fuse=$f cold $m"
  done
done
python -m pytest tests/test_gpu_wavefront.py -q -x 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench_m4.json 2> gpurun_out/bench_m4.err
python -c "import json; d=json.load(open('gpurun_out/bench_m4.json')); print('value %.4g ms/it %.4f frac %.3f clocks %s' % (d['value'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))"

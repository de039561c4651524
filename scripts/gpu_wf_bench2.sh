#!/bin/bash
# in-bench (power-capped) comparison of fuse depths at their default segment lengths
mkdir -p gpurun_out
for f in 2 3 2 3; do
  python bench.py --no-cpu-baseline --no-e2e --sor-fuse $f > gpurun_out/wfb2_${f}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/wfb2_${f}.json')); print('fuse=$f value %.4g ms/it %.4f clocks %s' % (d['value'], d['poisson_ms_per_iteration'], d['clocks']))"
done

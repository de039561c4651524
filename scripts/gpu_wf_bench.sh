#!/bin/bash
# in-bench (power-capped) comparison of stage counts and fuse depths
mkdir -p gpurun_out
for S in 2 3; do
  IBM_NVCC_DEFS="-DWF_NSTG=$S" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for f in 2 3; do
    python bench.py --no-cpu-baseline --no-e2e --sor-fuse $f > gpurun_out/wfb_${S}_${f}.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/wfb_${S}_${f}.json')); print('stg=$S fuse=$f value %.4g ms/it %.4f clocks %s' % (d['value'], d['poisson_ms_per_iteration'], d['clocks']))"
  done
done

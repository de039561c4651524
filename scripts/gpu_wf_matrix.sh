#!/bin/bash
# build-parameter matrix for the fused pass: cold micro-benchmark and in-bench (power-capped)
mkdir -p gpurun_out
for cfg in "4 2 2" "4 3 2" "3 3 3" "2 3 3" "3 2 2"; do
  set -- $cfg; B=$1; S=$2; F=$3
  IBM_NVCC_DEFS="-DWF_MINB=$B -DWF_NSTG=$S" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $F 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
  python bench.py --no-cpu-baseline --no-e2e --sor-fuse $F > gpurun_out/wfm.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/wfm.json')); print('minb=$B stg=$S fuse=$F cold %s bench value %.4g ms/it %.4f sm %s W %s' % ('$m', d['value'], d['poisson_ms_per_iteration'], d['clocks']['sm_mhz'], d['clocks']['power_w_median']))"
done

#!/bin/bash
TAG=${1:-r02j}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
grep -E "^(FAILED|E )" gpurun_out/pytest_${TAG}.log | head -20
MID_TB_CASES=3 timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}.json > gpurun_out/mid_tb_${TAG}.log 2>&1
python -c "
import json, sys
for r in json.load(open(sys.argv[1])):
    print(r['case'], {k: (round(v['us_per_it'], 2), v['tb_m_used'], v.get('phi_bitwise_equal')) for k, v in r.items() if k.startswith('tb')})
" gpurun_out/mid_tb_${TAG}.json
for defs in "" "-DWF_SHORT=1"; do
  IBM_NVCC_DEFS="$defs" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  for L in 128 256; do
    echo "defs=[$defs] L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
  done
done
python paper_2402_17337_b200/build.py --force > /dev/null 2>&1

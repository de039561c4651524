#!/bin/bash
# Mid-size grids (BJ configs[1]/[2] and the sweep's 1024^2..2048^2): parity, the resident
# temporally blocked solve (k_sor_tb) against the launched passes, ncu of k_sor_tb on M1 and
# the cylinder.  Usage (under gpurun): bash scripts/gpu_midgrid.sh TAG
TAG=${1:-mid}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_${TAG}.log 2>&1
tail -1 gpurun_out/pytest_${TAG}.log
timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}.json > gpurun_out/mid_tb_${TAG}.log 2>&1
python -c "
import json, sys
for r in json.load(open(sys.argv[1])):
    print(r['case'], {k: (round(v['us_per_it'], 2), v['tb_m_used'], v.get('phi_bitwise_equal')) for k, v in r.items() if k.startswith('tb')})
" gpurun_out/mid_tb_${TAG}.json
for C in M1 cyl; do
  ncu --set full --clock-control none --import-source on -k regex:k_sor_tb -s 1 -c 1 \
      -o gpurun_out/prof_tb_${C}_${TAG} -f python scripts/ncu_tb_case.py $C 400 > gpurun_out/ncu_tb_${C}_${TAG}.log 2>&1
done

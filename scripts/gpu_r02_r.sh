#!/bin/bash
# resident mid-grid solve with recomputed reciprocals (larger grids: 1024^2, M2) -- parity + timings
TAG=${1:-r02r}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_${TAG}.log 2>&1
tail -1 gpurun_out/pytest_${TAG}.log
timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}.json > gpurun_out/mid_tb_${TAG}.log 2>&1
python -c "
import json, sys
for r in json.load(open(sys.argv[1])):
    print(r['case'], {k: (round(v['us_per_it'], 2), v['tb_m_used'], v.get('phi_bitwise_equal')) for k, v in r.items() if k.startswith('tb')})
" gpurun_out/mid_tb_${TAG}.json

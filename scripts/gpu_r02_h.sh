#!/bin/bash
# resident mid-grid solve: rows per pass TB_R = 1, 2, 4 (de-interleaved shared layout)
TAG=${1:-r02h}
mkdir -p gpurun_out
for R in 1 2 4; do
  IBM_NVCC_DEFS="-DTB_R=$R" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cfg1 or cylinder or ragged or persistent" > gpurun_out/pytest_${TAG}_R$R.log 2>&1
  echo "R=$R $(tail -1 gpurun_out/pytest_${TAG}_R$R.log)"
  MID_TB_CASES=3 timeout 900 python scripts/mid_grid_tb.py gpurun_out/mid_tb_${TAG}_R$R.json > /dev/null 2>&1
  python -c "
import json, sys
for r in json.load(open(sys.argv[1]))[:3]:
    print(r['case'], {k: (round(v['us_per_it'], 2), v['tb_m_used'], v.get('phi_bitwise_equal')) for k, v in r.items() if k.startswith('tb')})
" gpurun_out/mid_tb_${TAG}_R$R.json
done

#!/bin/bash
# lag 1 / 2 x {per-update ownership masks, per-slot masks, per-slot masks with one hot chunk body}
TAG=${1:-r02y}
mkdir -p gpurun_out
IBM_LIB_VARIANT=sh1 IBM_WF_LAG=2 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "sh1 lag2 $(tail -1 gpurun_out/pytest_${TAG}.log)"
for V in "" sm1 sh1; do
  for LAG in 1 2; do
    for L in 128 256; do
      echo "V=$V LAG=$LAG L=$L $(IBM_LIB_VARIANT=$V IBM_WF_LAG=$LAG IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['200']['ms_per_it'])")" >> gpurun_out/mb_${TAG}.txt
    done
  done
done
cat gpurun_out/mb_${TAG}.txt
IBM_LIB_VARIANT=sh1 IBM_WF_LAG=2 ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_sh1_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf_${TAG}.log

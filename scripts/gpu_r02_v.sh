#!/bin/bash
# four columns per lane (128-column strips) with the scalar-coefficient MODE 3 vs the 2-column kernel
TAG=${1:-r02v}
mkdir -p gpurun_out
for V in "" cpl4; do
  IBM_LIB_VARIANT=$V python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}_$V.log 2>&1; echo "V=$V $(tail -1 gpurun_out/pytest_${TAG}_$V.log)"
  for L in 128 256; do
    echo "V=$V L=$L $(IBM_LIB_VARIANT=$V IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1)" >> gpurun_out/mb_${TAG}.txt
  done
  echo "V=$V bench $(IBM_LIB_VARIANT=$V python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ms/it %.4f frac %.3f clk %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))")" >> gpurun_out/mb_${TAG}.txt
done
IBM_LIB_VARIANT=cpl4 ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf4_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf4_${TAG}.log 2>&1
cat gpurun_out/mb_${TAG}.txt

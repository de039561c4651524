#!/bin/bash
# elect-issued TMA (uniform item): 8 vs 12 warps/SM, L = 128 / 256; cold micro-benchmark + short power-capped bench
TAG=${1:-r02u}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -1 gpurun_out/pytest_${TAG}.log
IBM_LIB_VARIANT=m12 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}_m12.log 2>&1; tail -1 gpurun_out/pytest_${TAG}_m12.log
for V in "" m12; do
  for L in 128 256; do
    echo "V=$V L=$L $(IBM_LIB_VARIANT=$V IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1)" >> gpurun_out/mb_${TAG}.txt
  done
  echo "V=$V bench $(IBM_LIB_VARIANT=$V python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ms/it %.4f frac %.3f clk %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))")" >> gpurun_out/mb_${TAG}.txt
done
cat gpurun_out/mb_${TAG}.txt

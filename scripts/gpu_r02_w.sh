#!/bin/bash
# persistent fused pass with cross-item TMA prefetch and host-built segment tables
TAG=${1:-r02w}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_${TAG}.log
for L in 64 128 256 512; do
  echo "L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1)" >> gpurun_out/mb_${TAG}.txt
done
echo "bench $(python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ms/it %.4f frac %.3f clk %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))")" >> gpurun_out/mb_${TAG}.txt
cat gpurun_out/mb_${TAG}.txt
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf_${TAG}.log

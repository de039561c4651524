#!/bin/bash
# half-sweep lag 1 vs 2 (one CTA per item, host-built segment tables); parity under both lags
TAG=${1:-r02x}
mkdir -p gpurun_out
for LAG in 1 2; do
  IBM_WF_LAG=$LAG python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}_$LAG.log 2>&1; echo "LAG=$LAG $(tail -1 gpurun_out/pytest_${TAG}_$LAG.log)"
  for L in 128 256; do
    echo "LAG=$LAG L=$L $(IBM_WF_LAG=$LAG IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['200']['ms_per_it'])")" >> gpurun_out/mb_${TAG}.txt
  done
  echo "LAG=$LAG bench $(IBM_WF_LAG=$LAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('ms/it %.4f frac %.3f clk %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))")" >> gpurun_out/mb_${TAG}.txt
done
cat gpurun_out/mb_${TAG}.txt
IBM_WF_LAG=2 ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_lag2_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf_${TAG}.log

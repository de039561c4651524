#!/bin/bash
# A/B of runtime or build variants of the fused Poisson pass (k_sor_wf) on one GPU:
# fused-pass parity tests, cold 8192^2 micro-benchmark at two segment lengths and a
# short power-capped bench line per variant.  A variant is a set of environment
# assignments, e.g. "IBM_WF_LAG=2", "IBM_WF_PERSIST=1", "IBM_LIB_VARIANT=m12" (a build
# variant from scripts/build_variants.py), or "" for the default.
# Usage (under gpurun): bash scripts/gpu_experiment.sh TAG "VARIANT1" "VARIANT2" ...
TAG=${1:-exp}; shift
mkdir -p gpurun_out
for V in "$@"; do
  echo "== variant [$V]"
  env $V timeout 600 python -m pytest tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
  tail -1 gpurun_out/pytest_${TAG}.log
  for L in ${ROWS:-128 256}; do
    echo "L=$L cold ms/iteration $(env $V IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['200']['ms_per_it'])")"
  done
  env $V timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bench ms/iteration %.4f frac %.3f clocks %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))"
done

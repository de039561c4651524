#!/bin/bash
# segment length L under the power cap: bench lines (5 timed steps of 10^4 iterations) with L fixed
for L in 0 128 256 512; do
  if [ $L = 0 ]; then V=""; else V="IBM_WF_ROWS=$L"; fi
  env $V timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('L=$L ms/iteration %.4f frac %.3f clocks %s' % (d['poisson_ms_per_iteration'], d['roofline']['frac'], d['clocks']))"
done

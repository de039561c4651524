#!/bin/bash
# SURVEY §8(d) cfg4(i) Poisson micro-benchmark (tolerance off, 20 warm-up, median of 5 x 200 iterations)
# at the sizes where HBM % is judged (4096^2, 8192^2) for the fused and the one-iteration pass
mkdir -p gpurun_out
for n in 4096 8192; do
  for f in 3 1; do
    timeout 300 python scripts/microbench_sor.py $n 1 60 $f 2>/dev/null | tail -1 >> gpurun_out/microbench_8d.jsonl
  done
done
cat gpurun_out/microbench_8d.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); p=d['protocol_8d']; print(d['n'], 'fuse', d['sor_fuse'], 'ms/it median %.4f  pass %.4f ms  pass GB/s %.0f' % (p['ms_per_it_median'], p['ms_per_pass'], p['pass_GBs']))"

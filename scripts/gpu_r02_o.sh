#!/bin/bash
# production-mesh omega check, Table-1/2 performance report (oracle_seq / oracle_omp / GPU), input-scaling sweep
TAG=${1:-r02o}
mkdir -p gpurun_out
for w in 1.97 1.985 1.99; do
  timeout 600 python scripts/production_diag.py --steps 60 --omega-p $w --out gpurun_out/prod_w${w}_${TAG}.json > gpurun_out/prod_w${w}_${TAG}.log 2>&1
  python -c "
import json, numpy as np, sys
d = json.load(open(sys.argv[1])); L = d['log']
its = [i for r in L for i in r['it_p']]
print('omega', sys.argv[2], 'steps', L[-1]['step'], 'status', L[-1]['status'], 'it_p mean (steps 21-60)', np.mean(its[20:]), 'max', max(its))
" gpurun_out/prod_w${w}_${TAG}.json $w
done
nproc; lscpu | grep -E "Model name|^CPU\(s\)" 
timeout 900 python scripts/perf_report.py --level 1 --maxit-p 200 --out gpurun_out/r02_perf_report > gpurun_out/perf_${TAG}.log 2>&1; tail -14 gpurun_out/perf_${TAG}.log
timeout 1200 python scripts/sweep_sizes.py --out gpurun_out/r02_sweep.json > gpurun_out/sweep_${TAG}.log 2>&1; cut -c1-250 gpurun_out/sweep_${TAG}.log

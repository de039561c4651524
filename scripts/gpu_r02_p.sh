#!/bin/bash
# fused-pass segment lengths incl. the wave-filling candidates, then the bench (online tuner over 6 candidates)
TAG=${1:-r02p}
mkdir -p gpurun_out
for L in 128 140 222 256 284 374; do
  echo "L=$L $(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 3 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*')"
done
python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms/step %.1f poisson ms/it %.4f frac %.3f e2e %.4g clocks %s' % (d['value'], d['ms_per_step'], d['poisson_ms_per_iteration'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))"
python -c "
import ibm_inputs as I, paper_2402_17337_b200 as P
cfg = I.cfg4(n=8192, maxit_p=400)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs()); g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny)); g.step(1); print('tuned L', g.query('wf_L'))"

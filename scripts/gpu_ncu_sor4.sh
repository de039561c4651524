#!/bin/bash
# full capture of a Poisson SOR launch on the state after 3 full 10^4-iteration steps
TAG=${1:-s}
mkdir -p gpurun_out
# launches before the micro-benchmark: per step ~13 velocity + 10000 pressure
ncu --set full --clock-control none --import-source on -k regex:k_sor -s 30050 -c 1 \
    -o gpurun_out/prof_sor3_${TAG} -f python scripts/microbench_sor.py 8192 3 10000 > gpurun_out/ncu_sor3_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_sor3_${TAG}.log
python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, ibm_inputs as I, paper_2402_17337_b200 as P
cfg = I.cfg4(n=8192, maxit_p=10000)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs()); g.set_body(*cfg.body_args()); g.set_fields(*I.initial_fields(cfg.nx, cfg.ny))
g.step(3)
phi = g.get("phi", device=True).abs()
for t in (0.0, 1e-300, 1e-280, 1e-250, 1e-200, 1e-100, 1e-20):
    print("frac |phi| <= %g : %.4f" % (t, float((phi <= t).double().mean())))
PY

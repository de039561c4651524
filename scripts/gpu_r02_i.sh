#!/bin/bash
TAG=${1:-r02i}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_wavefront.py -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
tail -2 gpurun_out/pytest_${TAG}.log
grep -E "^(FAILED|E )" gpurun_out/pytest_${TAG}.log | head -20
ncu --set full --clock-control none --import-source on -k regex:k_sor_tb -c 1 \
    -o gpurun_out/prof_tb_M1_${TAG} -f python -c "
import ibm_inputs as I, paper_2402_17337_b200 as P
cfg = I.cfg3(1, maxit_p=300)
g = P.Solver(cfg.xn, cfg.yn, **cfg.solver_kwargs()); g.set_body(*cfg.body_args())
g.set_fields(*I.initial_fields(cfg.nx, cfg.ny, 0.01)); g.step(1)
" > gpurun_out/ncu_tb_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_tb_${TAG}.log
python scripts/validate_cylinder.py --nx 1024 --ny 768 --dt 0.01 --steps 10000 --omega-p 1.95 --out gpurun_out/r02_cylinder_1024x768 > gpurun_out/cyl1024_${TAG}.log 2>&1
tail -c 1200 gpurun_out/cyl1024_${TAG}.log

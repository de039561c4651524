#!/bin/bash
TAG=${1:-r02k}
mkdir -p gpurun_out
IBM_WF_ROWS=256 ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf256_${TAG} -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf_${TAG}.log
timeout 900 python scripts/production_diag.py --steps 400 --out gpurun_out/prod_diag_${TAG}.json > gpurun_out/prod_diag_${TAG}.log 2>&1
tail -4 gpurun_out/prod_diag_${TAG}.log | cut -c1-400
timeout 1500 python scripts/validate_cylinder.py --nx 1024 --ny 768 --dt 0.01 --steps 8000 --omega-p 1.98 --maxit-p 30000 --out gpurun_out/r02_cylinder_1024x768 > gpurun_out/cyl1024_${TAG}.log 2>&1
tail -c 1500 gpurun_out/cyl1024_${TAG}.log

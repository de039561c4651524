#!/bin/bash
# ncu evidence for the per-step kernels (DRAM counters), the resident mid-grid solve
# (M1, cylinder) and the launch list of the bench command
TAG=${1:-r02z}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:'k_pred|k_prhs|k_correct|k_outlet|k_pext' -c 8 \
    -o gpurun_out/prof_step_${TAG} -f python bench.py --steps 1 --warmup 0 --maxit-p 5 --maxit-uv 3 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > gpurun_out/ncu_step_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_step_${TAG}.log
for C in M1 cyl; do
  ncu --set full --clock-control none --import-source on -k regex:k_sor_tb -s 1 -c 1 \
      -o gpurun_out/prof_tb_${C}_${TAG} -f python scripts/ncu_tb_case.py $C 400 > gpurun_out/ncu_tb_${C}_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_tb_${C}_${TAG}.log
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 0 --maxit-p 200 --no-e2e --no-cpu-baseline --no-clocks --sor-batch 256 > /dev/null 2>&1
wc -l gpurun_out/launches_${TAG}.csv

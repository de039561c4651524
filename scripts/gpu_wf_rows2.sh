#!/bin/bash
# fused-pass parity tests, then segment length L (IBM_WF_ROWS), default build (cold micro-benchmark)
mkdir -p gpurun_out
python paper_2402_17337_b200/build.py --force 2>&1 | grep -A2 "k_sor_wfILi3ELi0" | grep -o "Used [0-9]* registers"
timeout 600 python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for f in 3; do
  for L in 128 256 320; do
    m=$(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "fuse=$f L=$L cold $m"
  done
done
for f in 2; do
  for L in 66 132 258; do
    m=$(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "fuse=$f L=$L cold $m"
  done
done
for f in 4; do
  for L in 130 250; do
    m=$(IBM_WF_ROWS=$L timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "fuse=$f L=$L cold $m"
  done
done

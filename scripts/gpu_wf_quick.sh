#!/bin/bash
# fused-pass parity tests + cold micro-benchmark (m = 3 and 2), default build
mkdir -p gpurun_out
python paper_2402_17337_b200/build.py --force > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
grep -A2 "k_sor_wfILi3ELi0" gpurun_out/build.log | grep -o "Used [0-9]* registers"
timeout 600 python -m pytest tests/test_gpu_wavefront.py -q -x 2>&1 | tail -1
for f in ${FUSES:-3 2}; do
  m=$(timeout 300 python scripts/microbench_sor.py 8192 1 200 $f 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
  echo "fuse=$f cold $m"
done

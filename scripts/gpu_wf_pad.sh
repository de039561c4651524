#!/bin/bash
# row-pitch padding x segment length for the fused pass
mkdir -p gpurun_out
for PAD in 1 0; do
  for fl in "3 96" "3 128" "3 192" "3 256" "2 64" "2 96"; do
    set -- $fl
    m=$(IBM_PITCH_PAD=$PAD IBM_WF_ROWS=$2 timeout 300 python scripts/microbench_sor.py 8192 1 200 $1 2>&1 | tail -1 | grep -o '"200": {"ms_per_it": [0-9.]*' | grep -o '[0-9.]*$')
    echo "pad=$PAD fuse=$1 rows=$2 cold $m"
  done
done

#!/bin/bash
# ncu source capture of one fused pass for a build variant: gpu_ncu_wf_variant.sh TAG "DEFS" [FUSE]
TAG=$1; DEFS=$2; F=${3:-3}
mkdir -p gpurun_out
IBM_NVCC_DEFS="$DEFS" python paper_2402_17337_b200/build.py --force > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sor_wf -s 40 -c 1 \
    -o gpurun_out/prof_wf_${TAG} -f python scripts/microbench_sor.py 8192 1 120 $F > gpurun_out/ncu_wf_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_wf_${TAG}.log

#!/bin/bash
# two-warp pipeline (IBM_WF_WS=1): parity incl. the 8192^2 full-size case, A/B against the default, ncu
mkdir -p gpurun_out
IBM_WF_WS=1 timeout 900 python -m pytest tests/test_gpu_wavefront.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_ws.log 2>&1; tail -2 gpurun_out/pytest_ws.log
bash scripts/gpu_experiment.sh ws "" "IBM_WF_WS=1" "IBM_WF_WS=1 IBM_LIB_VARIANT=wsa" "IBM_WF_WS=1 IBM_LIB_VARIANT=wsc" 2>&1
IBM_WF_WS=1 ncu --set full --clock-control none --import-source on -k regex:k_sor_ws -s 40 -c 1 \
    -o gpurun_out/prof_ws2 -f python scripts/microbench_sor.py 8192 1 120 3 > gpurun_out/ncu_ws.log 2>&1
tail -1 gpurun_out/ncu_ws.log

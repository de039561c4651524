#!/bin/bash
# debug: peer-halo loopback cases (all), then compute-sanitizer on the failing one
TAG=${1:-r02ab}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_wavefront.py -k "peer_halo" -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; tail -15 gpurun_out/pytest_${TAG}.log
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_gpu_wavefront.py -k "test_loopback_peer_halo and 3-130-98-2-1" -x -q -p no:cacheprovider > gpurun_out/sanitizer_${TAG}.log 2>&1
grep -m 20 -A6 "Invalid\|Error\|error" gpurun_out/sanitizer_${TAG}.log | head -60

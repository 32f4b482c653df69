#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native_runtime.py -q > gpurun_out/pytest_native.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_native.log
bash tools/gpu_r2_ncu.sh

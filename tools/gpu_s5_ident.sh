#!/bin/bash
# Session 5: packed identity levels (u8 / u16) in the line kernels: parity suites + C3 / C2 ncu durations.
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 2400 python -m pytest tests/test_gpu_lines.py tests/test_gpu_lines2d.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_limits.py tests/test_gpu_cli.py tests/test_gpu_native_runtime.py -m gpu -q -x > $O/pytest_ident.log 2>&1; echo "rc=$?" >> $O/pytest_ident.log
bash tools/gpu_2d_ab2.sh; cp gpurun_out/ab2d.log $O/ab_lines2d_ident.log

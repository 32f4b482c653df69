#!/bin/bash
# Session 5: parity suite on the rebuilt map kernel, then A/B against variants (durations, shared wavefronts,
# ncu --set full summaries at C4a).
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 1500 python -m pytest tests/test_gpu_map3d.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_cli.py tests/test_gpu_distributed.py tests/test_gpu_native_runtime.py -m gpu -q -x > $O/pytest_map.log 2>&1; echo "rc=$?" >> $O/pytest_map.log
bash tools/gpu_s5_map2.sh "$@"

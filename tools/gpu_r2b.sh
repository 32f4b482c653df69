#!/bin/bash
# Round-2 visit B: new API / large-M tests, then the whole GPU suite (minus the slow config tests) and smoke.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_map2d.py tests/test_gpu_map3d.py -q > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log

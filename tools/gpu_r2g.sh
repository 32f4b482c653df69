#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log

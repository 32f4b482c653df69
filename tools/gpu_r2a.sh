#!/bin/bash
# Round-2 visit A: config-scale parity tests, the GPU suite, a bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q --durations=0 > gpurun_out/pytest_configs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_configs.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err

#!/bin/bash
# One gpurun visit: probe the box, GPU tests, smoke, microbench, benches.
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | head -20; } > gpurun_out/box.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 120 ./tools/ubench_atoms > gpurun_out/ubench_atoms.log 2>&1
timeout 600 python bench.py --config small --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_small.log 2>&1; echo "rc=$?" >> gpurun_out/bench_small.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log

#!/bin/bash
# One gpurun visit: GPU tests, smoke, microbench, timing, bench, ncu of the two 3D kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 120 ./tools/ubench_atoms > gpurun_out/ubench_atoms.log 2>&1
timeout 600 python tools/prof_run.py c5 4 both > gpurun_out/prof_c5.log 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 600 python tools/prof_run.py c4a 3 both > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lattice3d|hist3d_tiled" -s 2 -c 2 \
    -o gpurun_out/prof_v2 python tools/prof_run.py c4a 3 both > gpurun_out/ncu_v2.log 2>&1

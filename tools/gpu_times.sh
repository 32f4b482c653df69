#!/bin/bash
# Parity of the lines kernels + per-kernel durations (interior vs boundary) on C5 + timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lines.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
timeout 300 python tools/prof_run.py c5 3 lines > gpurun_out/prof_c5_lines.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lines3d --csv \
   --log-file gpurun_out/lines_times.csv python tools/prof_run.py c5 2 lines > gpurun_out/lines_times.log 2>&1

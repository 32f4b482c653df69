#!/bin/bash
# Lines kernel: parity, timing A/B against the lattice kernel, bench, ncu.
mkdir -p gpurun_out
timeout 120 ./tools/ubench_pipes > gpurun_out/ubench_pipes.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_lines.py tests/test_gpu_lattice.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
timeout 600 python tools/prof_run.py c5 4 all > gpurun_out/prof_c5_all.log 2>&1
timeout 600 python tools/prof_run.py c4a 4 all > gpurun_out/prof_c4a_all.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 1 \
    -o gpurun_out/prof_lines_c5 python tools/prof_run.py c5 2 lines > gpurun_out/ncu_lines.log 2>&1

#!/bin/bash
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none -k regex:lines3d -s 3 -c 1 \
    -o /tmp/ncu/prof_lines_boundary -f python tools/prof_run.py c5 2 lines > gpurun_out/ncu_lines_b.log 2>&1
ncu -i /tmp/ncu/prof_lines_boundary.ncu-rep --page raw --csv > gpurun_out/prof_lines_boundary_raw.csv 2>&1
ls -la /tmp/ncu >> gpurun_out/ncu_lines_b.log

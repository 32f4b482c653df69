#!/bin/bash
mkdir -p gpurun_out /tmp/ncu
FT_2D_KERNEL=lines timeout 300 python tools/prof_run.py c2 2 lattice > gpurun_out/plain_c2.log 2>&1 && \
FT_2D_KERNEL=lines timeout 600 ncu --set full --clock-control none --import-source on -k regex:lines2d -s 1 -c 1 \
    -o /tmp/ncu/prof_2d -f python tools/prof_run.py c2 2 lattice > gpurun_out/ncu_2d.log 2>&1
ncu -i /tmp/ncu/prof_2d.ncu-rep --page raw --csv > gpurun_out/prof_2d_raw.csv 2>&1
ncu -i /tmp/ncu/prof_2d.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_2d_sass.csv 2>&1

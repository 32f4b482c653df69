#!/bin/bash
# ncu --set full of the main lines kernel (2nd launch of the 2-rep run); raw CSV + source CSV written on the box.
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 1 \
    -o /tmp/ncu/prof_main -f python tools/prof_run.py c5 2 lines > gpurun_out/ncu_main.log 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page raw --csv > gpurun_out/prof_main_raw.csv 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_main_src.csv 2>&1

#!/bin/bash
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/prof_run.py c4a 2 map > gpurun_out/plain_map.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hist3d_tiled -s 1 -c 1 \
    -o /tmp/ncu/prof_map -f python tools/prof_run.py c4a 2 map > gpurun_out/ncu_map.log 2>&1
ncu -i /tmp/ncu/prof_map.ncu-rep --page raw --csv > gpurun_out/prof_map_raw.csv 2>&1

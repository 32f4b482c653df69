#!/bin/bash
# A/B of variants (args) + one full ncu capture of the main lines3d kernel with the source page.
mkdir -p gpurun_out /tmp/ncu
bash tools/gpu_ab.sh "$@"
timeout 300 python tools/prof_run.py c5 2 lines > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 1 \
    -o /tmp/ncu/prof_main -f python tools/prof_run.py c5 2 lines > gpurun_out/ncu_main.log 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page raw --csv > gpurun_out/prof_main_raw.csv 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page source --csv > gpurun_out/prof_main_source.csv 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_main_sass.csv 2>&1

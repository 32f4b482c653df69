#!/bin/bash
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/prof_run.py c4a 3 lines > gpurun_out/plain_c4a.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4a.csv python tools/prof_run.py c4a 3 lines > gpurun_out/ncu_c4a_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 1 \
    -o /tmp/ncu/prof_c4a -f python tools/prof_run.py c4a 3 lines > gpurun_out/ncu_c4a.log 2>&1
ncu -i /tmp/ncu/prof_c4a.ncu-rep --page raw --csv > gpurun_out/prof_c4a_raw.csv 2>&1
ncu -i /tmp/ncu/prof_c4a.ncu-rep --page details --csv > gpurun_out/prof_c4a_details.csv 2>&1

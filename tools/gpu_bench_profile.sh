#!/bin/bash
# Bench line + ncu launch list of the same command + one full ncu capture of the C5 lattice kernel.
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lattice|hist3d|curve_kernel|qmap" --csv \
    --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1
timeout 600 python tools/prof_run.py c5 2 lattice > gpurun_out/prof_plain_c5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice3d -s 1 -c 1 \
    -o gpurun_out/prof_c5 python tools/prof_run.py c5 2 lattice > gpurun_out/ncu_c5.log 2>&1

#!/bin/bash
# Kernel-only durations (ncu gpu__time_duration) of the 2D fused kernels on C2 / C3, both kernels.
mkdir -p gpurun_out
for c in c2 c3; do
  for k in lines lattice; do
    FT_2D_KERNEL=$k timeout 300 python tools/prof_run.py $c 3 lattice > gpurun_out/plain_${c}_${k}.log 2>&1 && \
    FT_2D_KERNEL=$k timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"lines2d|lattice2d" --csv \
        --log-file gpurun_out/ncu2d_${c}_${k}.csv python tools/prof_run.py $c 3 lattice > gpurun_out/ncu2d_${c}_${k}.log 2>&1
  done
done

#!/bin/bash
# 2D A/B: kernel durations (ncu) of ft_lines2d variants (FT_LIB) vs the main build, C2 and C3.
mkdir -p gpurun_out; rm -f gpurun_out/ab2d.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  for c in c2 c3; do
    FT_LIB=$lib FT_2D_KERNEL=lines timeout 300 python tools/prof_run.py $c 2 lattice > gpurun_out/plain_ab.log 2>&1 && \
    FT_LIB=$lib FT_2D_KERNEL=lines timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:lines2d --csv \
        --log-file gpurun_out/ab2d_${v}_${c}.csv python tools/prof_run.py $c 2 lattice > /dev/null 2>&1
    echo "$v $c $(grep -v '^==' gpurun_out/ab2d_${v}_${c}.csv | grep gpu__time | tail -1 | awk -F'","' '{print $NF}')" >> gpurun_out/ab2d.log
  done
done

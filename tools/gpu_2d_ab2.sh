#!/bin/bash
# 2D A/B: ncu kernel durations of ft_lines2d variants (FT_DEV_LIB, dev builds from tools/dev/variants.py) vs main, C2 and C3.
mkdir -p gpurun_out; rm -f gpurun_out/ab2d.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  for c in c2 c3; do
    FT_DEV_LIB=$lib timeout 300 python tools/prof_run.py $c 2 lattice > gpurun_out/plain_ab_${v}_${c}.log 2>&1 && \
    FT_DEV_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:lines2d --csv \
        --log-file gpurun_out/ab2d_${v}_${c}.csv python tools/prof_run.py $c 3 lattice > /dev/null 2>&1
    echo "$v $c $(grep -v '^==' gpurun_out/ab2d_${v}_${c}.csv | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')" >> gpurun_out/ab2d.log
  done
done

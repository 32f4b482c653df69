#!/bin/bash
# 3D A/B: ncu kernel durations + DRAM bytes of ft_lines3d variants (FT_DEV_LIB builds from tools/dev/variants.py)
# vs main, C5 and C4a; plain event timings too.  Every command under a hard timeout (a barrier bug would hang).
mkdir -p gpurun_out; rm -f gpurun_out/ab3d.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  for c in c5 c4a; do
    FT_DEV_LIB=$lib timeout -s KILL 300 python tools/prof_run.py $c 4 lines > gpurun_out/plain3_${v}_${c}.log 2>&1 || { echo "$v $c FAILED" >> gpurun_out/ab3d.log; continue; }
    FT_DEV_LIB=$lib timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:lines3d --csv \
        --log-file gpurun_out/ab3d_${v}_${c}.csv python tools/prof_run.py $c 2 lines > /dev/null 2>&1
    echo "$v $c $(grep -v '^==' gpurun_out/ab3d_${v}_${c}.csv | grep -E 'gpu__time|dram__bytes|lts__t_sectors' | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tr '\n' ' ')  | $(grep Gvox gpurun_out/plain3_${v}_${c}.log | tail -2 | tr '\n' ' ')" >> gpurun_out/ab3d.log
  done
done

#!/bin/bash
# Map-kernel A/B: ncu durations of hist3d_march in dev variants (FT_DEV_LIB) vs main, C5 and C4a.
mkdir -p gpurun_out; rm -f gpurun_out/abmap.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  for c in c5 c4a; do
    FT_DEV_LIB=$lib timeout -s KILL 300 python tools/prof_run.py $c 3 map > gpurun_out/plainm_${v}_${c}.log 2>&1 || { echo "$v $c FAILED" >> gpurun_out/abmap.log; continue; }
    FT_DEV_LIB=$lib timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:hist3d_march --csv \
        --log-file gpurun_out/abm_${v}_${c}.csv python tools/prof_run.py $c 2 map > /dev/null 2>&1
    echo "$v $c $(grep -v '^==' gpurun_out/abm_${v}_${c}.csv | grep -E 'gpu__time|wavefronts' | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tr '\n' ' ')" >> gpurun_out/abmap.log
  done
done

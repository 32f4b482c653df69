#!/bin/bash
# Session 5: parity of the byte-address 2D map kernel + A/B (ncu durations, C2 / C3) against variants.
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 1500 python -m pytest tests/test_gpu_map2d.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_cli.py tests/test_gpu_lines2d.py -m gpu -q -x > $O/pytest_map2d.log 2>&1; echo "rc=$?" >> $O/pytest_map2d.log
rm -f $O/ab_map2d.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  for c in c2 c3; do
    FT_DEV_LIB=$lib timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:hist2d_march --csv \
        --log-file $O/abm2d_${v}_${c}.csv python tools/prof_run.py $c 3 map > /dev/null 2>&1
    echo "$v $c $(grep -v '^==' $O/abm2d_${v}_${c}.csv | grep -E 'gpu__time|wavefronts' | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tr '\n' ' ')" >> $O/ab_map2d.log
  done
done

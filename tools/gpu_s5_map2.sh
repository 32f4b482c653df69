#!/bin/bash
# Session 5: map-kernel A/B (durations + shared wavefronts at C5 / C4a) and an ncu --set full summary of each
# variant at C4a.  Args: variant names under variants/.
mkdir -p gpurun_out/s5 /tmp/ncu
O=gpurun_out/s5
bash tools/gpu_map_ab.sh "$@"
cp gpurun_out/abmap.log $O/ab_map2.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  FT_DEV_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:hist3d_march -s 1 -c 1 \
      -o /tmp/ncu/map_$v -f python tools/prof_run.py c4a 2 map > /tmp/ncu/map_$v.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/map_$v.ncu-rep > $O/map_c4a_$v.summary.txt 2>&1
  ncu -i /tmp/ncu/map_$v.ncu-rep --page source --csv --print-source sass > /tmp/ncu/map_$v.sass.csv 2>&1
  python tools/ncu_sass_mix.py /tmp/ncu/map_$v.sass.csv > $O/map_c4a_$v.sassmix.txt 2>&1
done

#!/bin/bash
# Session 5: 2D line kernel A/B (ncu durations C2 / C3) + ncu --set full summaries at C2 of each variant.
mkdir -p gpurun_out/s5 /tmp/ncu
O=gpurun_out/s5
bash tools/gpu_2d_ab2.sh "$@"; cp gpurun_out/ab2d.log $O/ab_lines2d_b.log
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="variants/$v/libfieldtopo_b200.so"
  FT_DEV_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:lines2d -s 1 -c 1 \
      -o /tmp/ncu/l2d_$v -f python tools/prof_run.py c2 3 lattice > /tmp/ncu/l2d_$v.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/l2d_$v.ncu-rep > $O/lines2d_c2_$v.summary.txt 2>&1
done

#!/bin/bash
# Session 5: ncu --set full summaries of the kernels changed after the closing evidence (C4b line + map, C3 line, C3 map).
mkdir -p gpurun_out/s5caps /tmp/ncu
O=gpurun_out/s5caps
cap() {  # name cfg mode kernel-regex
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o /tmp/ncu/$1 -f python tools/prof_run.py $2 2 $3 > /tmp/ncu/$1.ncu.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$1.ncu-rep > $O/$1.summary.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass > /tmp/ncu/$1.sass.csv 2>&1
  python tools/ncu_sass_mix.py /tmp/ncu/$1.sass.csv > $O/$1.sassmix.txt 2>&1
}
cap lines3d_c4b c4b lines lines3d
cap hist3d_c4b c4b map hist3d_march
cap lines2d_c3 c3 lattice lines2d
cap hist2d_c3 c3 map hist2d_march

#!/bin/bash
# ncu --set full captures of every shipping hot kernel (one launch each, after
# the same command ran clean without ncu); summaries only come back (gpurun_out <= 64 MiB).
mkdir -p gpurun_out/ncu_r2 /tmp/ncu
O=gpurun_out/ncu_r2
cap() {  # name cfg mode kernel-regex
  timeout 600 python tools/prof_run.py $2 2 $3 > $O/$1.plain.log 2>&1 || { echo "plain run failed" >> $O/$1.plain.log; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o /tmp/ncu/$1 -f python tools/prof_run.py $2 2 $3 > $O/$1.ncu.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$1.ncu-rep > $O/$1.summary.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass > /tmp/ncu/$1.sass.csv 2>&1
  python tools/ncu_sass_mix.py /tmp/ncu/$1.sass.csv > $O/$1.sassmix.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > /tmp/ncu/$1.raw.csv 2>&1
  gzip -c /tmp/ncu/$1.raw.csv > $O/$1.raw.csv.gz
}
cap lines3d_c5 c5 lines lines3d
cap hist3d_c5 c5 map hist3d_march
cap hist3d_c4a c4a map hist3d_march
cap lines3d_c4b c4b lines lines3d
cap lines2d_c2 c2 lattice lines2d
cap lines2d_c3 c3 lattice lines2d
cap hist2d_c2 c2 map hist2d_march
du -sh /tmp/ncu > $O/du.txt

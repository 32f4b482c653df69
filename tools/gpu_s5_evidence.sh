#!/bin/bash
# Session-5 evidence: GPU suite, smoke, bench + reference arm, ncu launch list of the bench,
# event timings of every config, ncu --set full of every shipping hot kernel (summaries + SASS mix).
mkdir -p gpurun_out/s5g /tmp/ncu
O=gpurun_out/s5g
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
for c in c2 c3 c4a c4b c5; do timeout 600 python tools/prof_run.py $c 5 all > $O/prof_$c.log 2>&1; done
cap() {  # name cfg mode kernel-regex
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 \
      -o /tmp/ncu/$1 -f python tools/prof_run.py $2 2 $3 > /tmp/ncu/$1.ncu.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$1.ncu-rep > $O/$1.summary.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass > /tmp/ncu/$1.sass.csv 2>&1
  python tools/ncu_sass_mix.py /tmp/ncu/$1.sass.csv > $O/$1.sassmix.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > /tmp/ncu/$1.raw.csv 2>&1
  gzip -c /tmp/ncu/$1.raw.csv > $O/$1.raw.csv.gz
}
cap lines3d_c5 c5 lines lines3d
cap lines2d_c2 c2 lattice lines2d
cap lines2d_c3 c3 lattice lines2d
cap lines3d_c4b c4b lines lines3d
cap lines3d_c4a c4a lines lines3d
cap hist3d_c5 c5 map hist3d_march
cap hist2d_c2 c2 map hist2d_march

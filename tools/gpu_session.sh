#!/bin/bash
# One gpurun visit: GPU parity tests, smoke, bench line, ncu launch list of the
# bench command, one full ncu capture of the C5 main kernel (summarised on the box).
mkdir -p gpurun_out /tmp/ncu
python -c "from paper_2311_11740_b200 import build as b; print(\"lib up to date:\", b.up_to_date())" > gpurun_out/libcheck.log 2>&1
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/prof_run.py c5 3 all > gpurun_out/prof_c5.log 2>&1
timeout 600 python tools/prof_run.py c4a 3 all > gpurun_out/prof_c4a.log 2>&1
timeout 600 python tools/prof_run.py c4b 3 all > gpurun_out/prof_c4b.log 2>&1
timeout 600 python tools/prof_run.py c2 3 both > gpurun_out/prof_c2.log 2>&1
timeout 900 python tools/prof_run.py c3 3 both > gpurun_out/prof_c3.log 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lines|lattice|hist3d|curve_kernel|qmap" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 1 -c 1 \
    -o /tmp/ncu/prof_main -f python tools/prof_run.py c5 2 lines > gpurun_out/ncu_main.log 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page raw --csv > gpurun_out/prof_main_raw.csv 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page details --csv > gpurun_out/prof_main_details.csv 2>&1
ncu -i /tmp/ncu/prof_main.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_main_sass.csv 2>&1

#!/bin/bash
# One gpurun visit: GPU parity tests, smoke, bench line, ncu launch list of the
# bench command, one full ncu capture of the C5 lattice kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/prof_run.py c5 3 lattice > gpurun_out/prof_c5.log 2>&1
timeout 600 python tools/prof_run.py c2 3 lattice > gpurun_out/prof_c2.log 2>&1
timeout 600 python tools/prof_run.py c3 3 lattice > gpurun_out/prof_c3.log 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lattice|hist3d|curve_kernel|qmap" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice3d -s 1 -c 1 \
    -o gpurun_out/prof_c5 python tools/prof_run.py c5 2 lattice > gpurun_out/ncu_c5.log 2>&1

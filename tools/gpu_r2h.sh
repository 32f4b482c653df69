#!/bin/bash
# Session baseline: GPU parity suite, smoke, default bench line + reference arm, config kernel times.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in c2 c3 c4a c4b c5; do timeout 600 python tools/prof_run.py $c 5 all > gpurun_out/prof_$c.log 2>&1; done

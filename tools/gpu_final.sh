#!/bin/bash
# Closing visit: whole GPU suite, smoke, bench line + reference arm on the final code.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err

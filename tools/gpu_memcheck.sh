#!/bin/bash
# Lines parity + memcheck (one sanitizer tool) of the streaming tests, then the C5 bench.
mkdir -p gpurun_out
python -c "from paper_2311_11740_b200 import build as b; print(\"lib up to date:\", b.up_to_date())" > gpurun_out/libcheck.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lines.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_lines.py -x -q -k "streaming or column_tiles" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err

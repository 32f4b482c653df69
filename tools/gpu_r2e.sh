#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_map3d.py tests/test_gpu_map2d.py tests/test_gpu_parity.py tests/test_gpu_api.py -q > gpurun_out/pytest_map.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_map.log
for c in c5 c4a c4b c2 c3; do timeout 600 python tools/prof_run.py $c 3 map > gpurun_out/prof_map_$c.log 2>&1; done

#!/bin/bash
# Session 5: 3D map kernel with RP = 8 / 32 copies of the XOR-relative rank tables (no absolute-table march path):
# parity suites + event timings of the map kernel at C4b / C4a / C5.
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 2400 python -m pytest tests/test_gpu_map3d.py tests/test_gpu_limits.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_cli.py tests/test_gpu_native_runtime.py tests/test_gpu_distributed.py -m gpu -q -x > $O/pytest_rp.log 2>&1; echo "rc=$?" >> $O/pytest_rp.log
for c in c4b c4a c5; do timeout 300 python tools/prof_run.py $c 4 map > $O/prof_map_rp_$c.log 2>&1; done
timeout 600 python tools/gpu_fuzz.py 600 5 > $O/fuzz_rp.log 2>&1

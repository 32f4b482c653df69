#!/bin/bash
# Session 5: parity of the rebuilt map kernel (lane-replicated XOR-relative rank tables, FMA-pipe address
# arithmetic) + A/B against the previous build (variants/mapold).
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 1500 python -m pytest tests/test_gpu_map3d.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_configs.py tests/test_gpu_cli.py tests/test_gpu_distributed.py tests/test_gpu_native_runtime.py -m gpu -q -x > $O/pytest_map.log 2>&1; echo "rc=$?" >> $O/pytest_map.log
bash tools/gpu_map_ab.sh "$@"
cp gpurun_out/abmap.log $O/ab_map.log
cat gpurun_out/plainm_*_c5.log > $O/plain_c5.log

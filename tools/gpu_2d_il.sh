#!/bin/bash
# 2D interleaved-warp work split: A/B vs the previous split (variants/prev2d) + 2D parity tests.
mkdir -p gpurun_out/s4
O=gpurun_out/s4
timeout 900 python -m pytest tests/test_gpu_lines2d.py tests/test_gpu_configs.py tests/test_gpu_api.py -m gpu -q -k "lines2d or config2 or config3 or batch or 2d" > $O/pytest_2d.log 2>&1; echo "rc=$?" >> $O/pytest_2d.log
bash tools/gpu_2d_ab2.sh prev2d
cp gpurun_out/ab2d.log $O/ab_lines2d_il.log
for v in main prev2d; do for c in c2 c3; do cat gpurun_out/ab2d_${v}_${c}.csv | grep -v '^==' | grep dram__bytes >> $O/ab_lines2d_il_dram.log; done; done

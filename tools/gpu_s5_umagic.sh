#!/bin/bash
# Session 5: the exact integer u8/u16 decoding in ft_lines3d (FT_Q_UMAGIC): exhaustive quantizer tests, line /
# config / API / parity suites, C4b timings (events + ncu).
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 2400 python -m pytest tests/test_gpu_quant_exhaustive.py tests/test_gpu_lines.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_native_runtime.py tests/test_gpu_distributed.py tests/test_gpu_cli.py -m gpu -q -x > $O/pytest_umagic.log 2>&1; echo "rc=$?" >> $O/pytest_umagic.log
timeout 300 python tools/prof_run.py c4b 5 lines > $O/prof_c4b_umagic.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lines3d --csv --log-file $O/ncu_c4b_umagic.csv python tools/prof_run.py c4b 3 lines > /dev/null 2>&1

#!/bin/bash
# Session 5: parity of the line kernels on the mirrored shared layout (IDP.2A select + split), then A/B
# against the previous build (variants/lprev): ncu durations C5 / C4a (3D) and C2 / C3 (2D).
mkdir -p gpurun_out/s5
O=gpurun_out/s5
timeout 1800 python -m pytest tests/test_gpu_lines.py tests/test_gpu_lines2d.py tests/test_gpu_lattice.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_native_runtime.py tests/test_gpu_distributed.py -m gpu -q -x > $O/pytest_lines.log 2>&1; echo "rc=$?" >> $O/pytest_lines.log
bash tools/gpu_3d_ab.sh "$@"; cp gpurun_out/ab3d.log $O/ab_lines3d_mirror.log
bash tools/gpu_2d_ab2.sh "$@"; cp gpurun_out/ab2d.log $O/ab_lines2d_mirror.log

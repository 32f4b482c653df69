#!/bin/bash
# A/B of ft_lines variants (FT_LIB) on C5 + parity tests on the main build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lines.py tests/test_gpu_lattice.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab.log
  FT_LIB=variants/$v/libfieldtopo_b200.so timeout 300 python tools/prof_run.py c5 4 lines 2>&1 | grep -v "rep 0" >> gpurun_out/ab.log
done
timeout 300 python tools/prof_run.py c5 4 lines 2>&1 | grep -v "rep 0" >> gpurun_out/ab.log

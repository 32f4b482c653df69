#!/bin/bash
# A/B of ft_lines variants (FT_LIB) on C5 + parity tests on the main build + ncu of the main build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lines.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
echo "== main" >> gpurun_out/ab.log
timeout 300 python tools/prof_run.py c5 3 lines 2>&1 | grep -v "rep 0" >> gpurun_out/ab.log
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab.log
  FT_LIB=variants/$v/libfieldtopo_b200.so timeout 300 python tools/prof_run.py c5 3 lines 2>&1 | grep -v "rep 0" >> gpurun_out/ab.log
done
#timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 2 \
#    -o python tools/prof_run.py c5 2 lines > gpurun_out/ncu_lines.log 2>&1
if [ -n "$NCU_VARIANT" ]; then
  FT_LIB=variants/$NCU_VARIANT/libfieldtopo_b200.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:lines3d -s 2 -c 1 \
    -o gpurun_out/prof_lines_$NCU_VARIANT python tools/prof_run.py c5 2 lines > gpurun_out/ncu_lines.log 2>&1
fi

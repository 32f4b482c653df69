#!/bin/bash
# lines parity + C5 / C4a / C4b kernel times
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
python -c "from paper_2311_11740_b200 import build as b; print(\"lib up to date:\", b.up_to_date())" > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lines.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
for cfg in c5 c4a c4b; do
  echo "== main $cfg" >> gpurun_out/ab.log
  timeout 300 python tools/prof_run.py $cfg 4 lines >> gpurun_out/ab.log 2>&1
done

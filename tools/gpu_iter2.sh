#!/bin/bash
# Iteration visit: lines parity, C5/C4a timing, dram bytes of the main kernel (ncu, 2 metrics).
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
python -c "from paper_2311_11740_b200 import build as b; print(\"lib up to date:\", b.up_to_date())" > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_lines.py -x -q > gpurun_out/pytest_lines.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lines.log
for cfg in c5 c4a; do
  echo "== main $cfg" >> gpurun_out/ab.log
  timeout 300 python tools/prof_run.py $cfg 4 lines >> gpurun_out/ab.log 2>&1
done
timeout 300 python tools/prof_run.py c5 2 lines > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lines3d --csv \
    --log-file gpurun_out/dram.csv python tools/prof_run.py c5 2 lines > gpurun_out/ncu_dram.log 2>&1

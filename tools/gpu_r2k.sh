#!/bin/bash
# Round-2 session-4 baseline visit: 2D tile-load microbenchmark (timing + ncu DRAM bytes),
# GPU suite, smoke, bench line.
mkdir -p gpurun_out/s4
O=gpurun_out/s4
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_tiles tools/ubench_tiles.cu > $O/ubench_build.log 2>&1
timeout 120 /tmp/ubench_tiles > $O/ubench_tiles.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:stream_tiles --csv --log-file $O/ubench_tiles_ncu.csv /tmp/ubench_tiles > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu_all.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_all.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err

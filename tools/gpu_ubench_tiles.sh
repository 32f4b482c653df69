#!/bin/bash
# 2D tile-load microbenchmark: timing + ncu DRAM bytes / L2 hit rate per variant.
mkdir -p gpurun_out/s4
O=gpurun_out/s4
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_tiles tools/ubench_tiles.cu > $O/ubench_build.log 2>&1
timeout 120 /tmp/ubench_tiles > $O/ubench_tiles2.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none \
    -k regex:stream_tiles --csv --log-file $O/ubench_tiles2_ncu.csv /tmp/ubench_tiles > /dev/null 2>&1

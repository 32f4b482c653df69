#!/bin/bash
# Round-2 visit C: distributed entry points on the GPU, streaming tests, C5s, ws=2 gloo plumbing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -q > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 900 python -m pytest tests -m gpu -q -k "stream or lowmem or lines or raw" --deselect tests/test_gpu_configs.py > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
timeout 900 python bench.py --config c5s --steps 2 --warmup 3 > gpurun_out/bench_c5s.json 2> gpurun_out/bench_c5s.err; echo "rc=$?" >> gpurun_out/bench_c5s.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c4a --dist-backend gloo --steps 3 --warmup 3 > gpurun_out/bench_ws2.json 2> gpurun_out/bench_ws2.err; echo "rc=$?" >> gpurun_out/bench_ws2.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err

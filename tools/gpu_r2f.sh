#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py -q > gpurun_out/pytest_api.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_api.log
timeout 900 python tools/stream_probe.py > gpurun_out/stream_probe.json 2> gpurun_out/stream_probe.err; echo "rc=$?" >> gpurun_out/stream_probe.err

mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_lines2d.py tests/test_gpu_configs.py tests/test_gpu_api.py tests/test_gpu_cli.py -q -x -k "not config5 and not config4" > gpurun_out/pytest_2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_2d.log
bash tools/gpu_2d_ab2.sh prev

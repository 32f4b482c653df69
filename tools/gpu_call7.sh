mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_lines.py tests/test_gpu_lattice.py tests/test_gpu_configs.py tests/test_gpu_api.py -q -x > gpurun_out/pytest_l3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l3.log
bash tools/gpu_3d_ab.sh

set -x
timeout 2400 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_reacting_loop.py tests/test_gpu_rom.py -q -rf > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
tail -n 3 gpurun_out/pytest_v.log

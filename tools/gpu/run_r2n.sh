set -x
timeout 1200 python -m pytest tests/test_gpu_rom.py tests/test_gpu_factored.py tests/test_gpu_bigsample.py tests/test_gpu_parity_configs.py -q -rf -k "not cfg3_recipe_200" > gpurun_out/pytest_n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.log
ADROM_QDEIM_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_n.log 2>&1
ADROM_QDEIM_RADIX=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_n_radix.log 2>&1
tail -n 2 gpurun_out/pytest_n.log

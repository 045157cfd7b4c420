set -x
timeout 1200 python -m pytest tests/test_gpu_core.py tests/test_gpu_dense_rules.py tests/test_gpu_rom.py -q -rf > gpurun_out/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.log
timeout 300 python tools/residual_bench.py > gpurun_out/residual_bench2.log 2>&1
timeout 900 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/bench_m_cfg1.log 2>&1
tail -n 2 gpurun_out/pytest_m.log; cat gpurun_out/residual_bench2.log

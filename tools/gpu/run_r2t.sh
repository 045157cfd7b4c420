set -x
timeout 900 python -m pytest tests/test_gpu_core.py -q -rf -k "sod or Sod or residual or newton" > gpurun_out/pytest_t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t.log
timeout 300 python tools/residual_bench.py > gpurun_out/residual_bench3.log 2>&1
tail -n 2 gpurun_out/pytest_t.log; cat gpurun_out/residual_bench3.log

set -x
timeout 1200 python -m pytest tests/test_gpu_isvd_core.py tests/test_gpu_core.py tests/test_gpu_factored.py -q -rf > gpurun_out/pytest_r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r.log
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --warmup 1900 --steps 20 > gpurun_out/bench_r_late.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --e2e-steps 2000 > gpurun_out/bench_r_e2e2000.log 2>&1
tail -n 2 gpurun_out/pytest_r.log
for f in gpurun_out/bench_r_late.log gpurun_out/bench_r_e2e2000.log; do tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], (d.get('e2e') or {}).get('value'))"; done

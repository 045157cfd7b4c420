# Round-2 check 3: new dense/rule tests, cfg4 bisection across commits, cfg3 parity diagnostics
set -x
timeout 1200 python -m pytest tests/test_gpu_dense_rules.py tests/test_gpu_dgemm.py -q -rf > gpurun_out/pytest_rules.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rules.log
for c in 2b84e3a f25eec0 8b3d57a; do
  (cd bisect/$c && timeout 600 python bench.py --config cfg4 --no-cpu-baseline > ../../gpurun_out/bisect_$c.log 2>&1)
done
timeout 900 python tests/cfg3_parity.py --n 65536 --steps 200 --envelope 2 > gpurun_out/cfg3_diag.log 2>&1
tail -n 2 gpurun_out/pytest_rules.log

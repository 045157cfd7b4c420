# Round-2 check 4: dense/rule tests after fixes, cfg3 pinned-decision diagnostics, cfg2 batch diag
set -x
timeout 1200 python -m pytest tests/test_gpu_dense_rules.py -q -rf > gpurun_out/pytest_rules2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rules2.log
timeout 1500 python tools/cfg3_pinned_diag.py > gpurun_out/cfg3_pinned.log 2>&1
timeout 900 python bench.py --config cfg2 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2b.log 2>&1
tail -n 2 gpurun_out/pytest_rules2.log

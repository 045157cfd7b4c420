set -x
timeout 2400 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_l.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_l.log 2>&1
for c in cfg0 cfg1 cfg2; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_l_$c.log 2>&1; done
tail -n 2 gpurun_out/pytest_l.log

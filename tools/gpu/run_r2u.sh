set -x
timeout 2400 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_u.log 2>&1
for c in cfg0 cfg1 cfg4; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_u_$c.log 2>&1; done
tail -n 2 gpurun_out/pytest_u.log
for f in gpurun_out/bench_u*.log; do tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['probes_ms_per_launch'].get('rom_step'))"; done

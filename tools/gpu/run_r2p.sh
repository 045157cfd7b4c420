set -x
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --warmup 1000 --steps 20 > gpurun_out/bench_p_late1000.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --warmup 1900 --steps 20 > gpurun_out/bench_p_late1900.log 2>&1
for f in gpurun_out/bench_p_late*.log; do tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['qdeim_rounds_per_step'], d['rom_iterations_mean'], d['probes_ms_per_launch'])"; done

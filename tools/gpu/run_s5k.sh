python -m pytest tests/test_gpu_factored.py tests/test_gpu_rom.py -m gpu -x -q > gpurun_out/s5k_test.log 2>&1; tail -2 gpurun_out/s5k_test.log
for w in 3 1000; do
timeout 900 python bench.py --steps 450 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/s5k_bench_w$w.log 2> gpurun_out/s5k_bench_w$w.err
tail -1 gpurun_out/s5k_bench_w$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup $w', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch']['qdeim_round'], d['probes_launches']['qdeim_round'], d['probes_launches']['isvd_reanchor'], d['probed_steps']['ms_per_step'], d['event_errors'])"
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch']['qdeim_round'])"

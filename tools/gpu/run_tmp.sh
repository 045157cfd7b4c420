python -m pytest tests/test_gpu_rom.py tests/test_gpu_factored.py -m gpu -x -q > gpurun_out/tmp_test.log 2>&1; tail -1 gpurun_out/tmp_test.log
for w in 3 1100; do
timeout 600 python bench.py --steps 60 --warmup $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup $w', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch']['qdeim_round'], d['event_errors'])"
done

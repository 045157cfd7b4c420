python -m pytest tests/test_gpu_factored.py tests/test_gpu_rom.py -m gpu -x -q > gpurun_out/s5t_test.log 2>&1; tail -1 gpurun_out/s5t_test.log
for w in 3 1100; do
timeout 600 python bench.py --steps 60 --warmup $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup $w', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch']['qdeim_round'], d['event_errors'])"
done
for c in cfg1 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/s5_bench_$c.log 2> gpurun_out/s5_bench_$c.err
  tail -1 gpurun_out/s5_bench_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c', d['value'], d['unit'], 'e2e', d.get('e2e'), 'roof', d.get('roofline',{}).get('frac'), d.get('roofline',{}).get('kernel','')[:60], 'probed', d.get('probed_steps'))"
done

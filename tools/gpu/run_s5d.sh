timeout 900 python bench.py --steps 950 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5d_bench2000.log 2> gpurun_out/s5d_bench2000.err
tail -1 gpurun_out/s5d_bench2000.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench2000', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch'], d['probes_launches'], d['event_errors'])"

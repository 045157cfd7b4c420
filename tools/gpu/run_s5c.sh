timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5c_bench.log 2> gpurun_out/s5c_bench.err
tail -1 gpurun_out/s5c_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch'], d['event_errors'])"
python -m pytest tests -m gpu -x -q > gpurun_out/s5c_gputest.log 2>&1; tail -3 gpurun_out/s5c_gputest.log

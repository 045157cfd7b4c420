python -m pytest tests/test_gpu_factored.py tests/test_gpu_rom.py -m gpu -x -q > gpurun_out/s5p_test.log 2>&1; tail -1 gpurun_out/s5p_test.log
for w in 3 1100; do
timeout 600 python bench.py --steps 60 --warmup $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup $w', d['value'], d['qdeim_rounds_per_step'], d['probes_ms_per_launch']['qdeim_round'], d['event_errors'])"
done
export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_c3_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/s5_c3_launches.csv 45 > gpurun_out/s5_c3_launch_summary.txt
head -12 gpurun_out/s5_c3_launch_summary.txt; tail -1 gpurun_out/s5_c3_launch_summary.txt

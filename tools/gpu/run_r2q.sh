set -x
export ADROM_PROFILE_TIMED=1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_late_timed.csv python bench.py --warmup 1900 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_late.log 2>&1
unset ADROM_PROFILE_TIMED
ADROM_QDEIM_TRACE=1 timeout 900 python bench.py --warmup 1900 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_q_trace.log 2>&1
grep "qdeim:" gpurun_out/bench_q_trace.log | tail -12

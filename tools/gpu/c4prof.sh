set -x
export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/c4_launches.csv python bench.py --config cfg4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4_ncu.log 2>&1
python tools/launches.py gpurun_out/c4_launches.csv 30 > gpurun_out/c4_launch_summary.txt
cat gpurun_out/c4_launch_summary.txt

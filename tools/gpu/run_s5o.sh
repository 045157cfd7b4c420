export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_c3_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/s5_c3_launches.csv 45 > gpurun_out/s5_c3_launch_summary.txt
cat gpurun_out/s5_c3_launch_summary.txt
grep "qp_refresh_bf" gpurun_out/s5_c3_launches.csv | awk -F'","' '{print $NF}' | head -12

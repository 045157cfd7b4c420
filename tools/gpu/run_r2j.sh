# Round-2 full validation: GPU suite, smoke, benches, timed launch lists, ncu captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke3.log
timeout 900 python bench.py > gpurun_out/bench3.log 2>&1
for c in cfg0 cfg1 cfg2 cfg4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench3_$c.log 2>&1; done
export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_timed.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_timed.csv python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:dmma_tn_kernel|rot_tc_kernel|bl_dir_kernel" -c 4 -o gpurun_out/c4_full python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4_full.log 2>&1
python tools/profile_summary.py full gpurun_out/c4_full.ncu-rep gpurun_out/c4_full.txt c4_full >> gpurun_out/ncu_c4_full.log 2>&1
tail -n 2 gpurun_out/pytest_full.log gpurun_out/smoke3.log

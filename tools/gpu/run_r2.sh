# Round-2 validation: GPU tests, smoke, cfg3 bench + reference arm, launch list, xpass ncu capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
for c in cfg2 cfg0 cfg1 cfg4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
export ADROM_PROFILE_TIMED=1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:xpass_tma" -c 2 -o gpurun_out/xpass_tma python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
python tools/profile_summary.py full gpurun_out/xpass_tma.ncu-rep gpurun_out/xpass_tma.txt xpass_tma >> gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/*.log

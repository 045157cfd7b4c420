set -x
export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:bl_dir|part_solve_tc|reacting_jac|lspg_update|bl_decode" -c 5 -o gpurun_out/c4_full python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
unset ADROM_PROFILE_TIMED
timeout 600 ncu --set full --clock-control none -k "regex:sod_rhs|burgers_rhs|reacting_rhs" -c 3 -o gpurun_out/res_full python tools/residual_bench.py > /dev/null 2>&1
python tools/profile_summary.py full gpurun_out/c4_full.ncu-rep gpurun_out/c4_full.txt "cfg4 kernels"
python tools/profile_summary.py full gpurun_out/res_full.ncu-rep gpurun_out/res_full.txt "residual kernels"
ls -la gpurun_out/

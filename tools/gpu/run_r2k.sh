# Round-2: ncu of the one-block kernels on the cfg3 critical path; full-N step parity prefix
set -x
export ADROM_PROFILE_TIMED=1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:lspg_kernel|isvd_core_kernel|qp_refresh_bf_kernel|qp_greedy_kernel" -c 4 -o gpurun_out/c3_oneblock python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_oneblock.log 2>&1
python tools/profile_summary.py full gpurun_out/c3_oneblock.ncu-rep gpurun_out/c3_oneblock.txt c3_oneblock >> gpurun_out/ncu_c3_oneblock.log 2>&1
ncu -i gpurun_out/c3_oneblock.ncu-rep --page source --csv --print-source sass -k regex:lspg_kernel > gpurun_out/c3_lspg_source.csv 2>/dev/null
unset ADROM_PROFILE_TIMED
timeout 300 python tools/residual_bench.py > gpurun_out/residual_bench.log 2>&1
timeout 2400 python tools/cfg3_fulln_prefix.py --steps 3 --out gpurun_out/c3_fulln.json > gpurun_out/c3_fulln.log 2>&1
tail -n 5 gpurun_out/c3_fulln.log

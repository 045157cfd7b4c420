# final profiles of this session (cfg 3): launch list of the timed region, ncu --set full of the QDEIM kernels
set -x
export ADROM_PROFILE_TIMED=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_c3_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/s5_c3_launches.csv gpurun_out/s5_c3_timed_launches.txt "round 2 (final): cfg3 adaptive-ROM loop, timed region only (10 steps, one event each), serialised"
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:qs_select_compact|qp_complement|qp_refresh_bf|qp_greedy|qp_resvec" -c 14 -o gpurun_out/s5_qdeim_final python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_qdeim_final.log 2>&1
python tools/profile_summary.py full gpurun_out/s5_qdeim_final.ncu-rep gpurun_out/s5_qdeim_final.txt "round 2 (final): QDEIM kernels of one cfg-3 event (selection, complement basis, refresh, residual vectors, greedy)"
unset ADROM_PROFILE_TIMED
for c in cfg0 cfg1 cfg2 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/s5_bench_$c.log 2> gpurun_out/s5_bench_$c.err
  tail -1 gpurun_out/s5_bench_$c.log | cut -c1-400
done

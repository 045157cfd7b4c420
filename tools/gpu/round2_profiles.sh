# The commands behind the round-2 evidence in profiles/ (run under gpurun on one B200).
set -x
export ADROM_PROFILE_TIMED=1
# launch list of the cfg-3 timed region -> profiles/r2_cfg3_timed_launches_final.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/c3_launches.csv gpurun_out/r2_cfg3_timed_launches_final.txt "round 2 (final): cfg3 adaptive-ROM loop, timed region only (10 steps, one event each), serialised"
# ncu --set full of the QDEIM kernels of one event -> profiles/r2_qdeim_kernels_full.txt
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:qs_select_compact|qp_complement|qp_refresh_bf|qp_greedy|qp_resvec" -c 14 -o gpurun_out/qdeim_final python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/qdeim_final.log 2>&1
python tools/profile_summary.py full gpurun_out/qdeim_final.ncu-rep gpurun_out/r2_qdeim_kernels_full.txt "round 2 (final): QDEIM kernels of one cfg-3 event"
# the basis passes (the bench's roofline kernels) -> profiles/r2_xpass_tma_full.txt, profiles/traffic.json
bash tools/gpu/ncu_full.sh "xpass_tma" xpass_tma_full 4 -- --steps 3 --warmup 3
unset ADROM_PROFILE_TIMED
# early / late windows of the 2000-step run -> profiles/r2_cfg3_long_run.txt
for w in 3 1000; do
  timeout 900 python bench.py --steps 450 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/long_w$w.log 2>&1
  tail -1 gpurun_out/long_w$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup $w', d['value'], d['qdeim_rounds_per_step'], d['probes_launches'].get('isvd_reanchor'), d['probed_steps'])"
done
# per-round trace (certified prefix, bound statistics)
ADROM_QDEIM_TRACE=2 timeout 600 python bench.py --steps 4 --warmup 1100 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/qdeim_trace.err

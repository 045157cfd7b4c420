set -x
ADROM_QDEIM_TRACE=1 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_trace.log 2> gpurun_out/s5_trace.err
grep -c "qdeim round" gpurun_out/s5_trace.err
bash tools/gpu/ncu_full.sh "qp_refresh_bf|qp_greedy|qp_resvec|qs_hist|qs_compact|gather_rows_tc" s5_qdeim_full 24 -- --steps 3 --warmup 3

set -x
timeout 1200 python bench.py --no-cpu-baseline --e2e-steps 2000 > gpurun_out/bench_o_e2e2000.log 2>&1
tail -n 1 gpurun_out/bench_o_e2e2000.log | cut -c1-300

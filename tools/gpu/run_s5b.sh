ADROM_QDEIM_TRACE=2 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_trace2.log 2> gpurun_out/s5_trace2.err
grep -A1 "qdeim round" gpurun_out/s5_trace2.err | tail -40

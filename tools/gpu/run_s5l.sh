ADROM_QDEIM_TRACE=2 timeout 900 python bench.py --steps 12 --warmup 1100 --no-cpu-baseline --no-e2e > gpurun_out/s5l.log 2> gpurun_out/s5l.err
grep -v "qdeim refresh:" gpurun_out/s5l.err | tail -n 60 > gpurun_out/s5l_tail.err

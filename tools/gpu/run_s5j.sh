ADROM_QDEIM_TRACE=2 timeout 900 python bench.py --steps 30 --warmup 1100 --no-cpu-baseline --no-e2e > gpurun_out/s5j.log 2> gpurun_out/s5j.err
grep -v "qdeim refresh:" gpurun_out/s5j.err | tail -n 150 > gpurun_out/s5j_tail.err

ADROM_QDEIM_TRACE=1 timeout 900 python bench.py --steps 100 --warmup 1100 --no-cpu-baseline --no-e2e > gpurun_out/s5i.log 2> gpurun_out/s5i.err
grep -c "qdeim: n=" gpurun_out/s5i.err
tail -n 400 gpurun_out/s5i.err > gpurun_out/s5i_tail.err

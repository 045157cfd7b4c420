for v in base lp8 lp32; do
  if [ $v = base ]; then cp build/variants/base.so paper_2605_28684_b200/lib/libadrom_b200.so; else cp build/variants/$v/libadrom_b200.so paper_2605_28684_b200/lib/libadrom_b200.so; fi
  timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>&1
  tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['probes_ms_per_launch']['isvd_core'])"
done

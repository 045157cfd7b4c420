for m in 32768 65536; do
  for f in 64 96 128 192; do
    for w in 3 1100; do
      ADROM_QDEIM_POOL_M=$m ADROM_QDEIM_REFRESH=$f timeout 600 python bench.py --steps 60 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
      tail -n 1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('M', $m, 'F', $f, 'warmup', $w, d['value'], 'rounds', d['qdeim_rounds_per_step'], 'round_ms', d['probes_ms_per_launch']['qdeim_round'])" >> gpurun_out/s5m_sweep.txt 2>&1
    done
  done
done
cat gpurun_out/s5m_sweep.txt

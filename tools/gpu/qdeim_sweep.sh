# QDEIM pool size / refresh factor sweep on the cfg-3 bench (device-timed, no e2e)
for m in 16384 32768 65536 131072; do
  for f in 64 128 256; do
    ADROM_QDEIM_POOL_M=$m ADROM_QDEIM_REFRESH=$f timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.log 2>&1
    tail -n 1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('M', $m, 'F', $f, d['value'], 'rounds', d['qdeim_rounds_per_step'], 'round_ms', d['probes_ms_per_launch']['qdeim_round'])" >> gpurun_out/qdeim_sweep.txt 2>&1
  done
done
cat gpurun_out/qdeim_sweep.txt

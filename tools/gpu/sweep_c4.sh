for S in 148 74 296; do for U in 512 1024 256; do
  ADROM_SPLITK=$S ADROM_UPD_THREADS=$U timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>&1
  tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splitk', $S, 'upd', $U, d['value'], d['probes_ms_per_launch']['rom_step'])"
done; done

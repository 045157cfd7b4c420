set -x
ADROM_DEFECT_N=65536 timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_2p16_ref.log 2>&1
ADROM_DEFECT_N=65536 ADROM_FACTORED=1 timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_2p16_fact_ref.log 2>&1
timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_2p24_ref.log 2>&1
grep step gpurun_out/cfg3_defect_*_ref.log
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_x.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_x.log 2>&1
tail -n 3 gpurun_out/pytest_x.log
tail -n 1 gpurun_out/bench_x.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"

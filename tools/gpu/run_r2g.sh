set -x
(cd bisect/head_oldcore && ADROM_CORE_OLD=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline > ../../gpurun_out/c4_head_oldcore.log 2>&1)
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py -q -rf -k cfg3 > gpurun_out/pytest_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cfg3.log
tail -n 3 gpurun_out/pytest_cfg3.log

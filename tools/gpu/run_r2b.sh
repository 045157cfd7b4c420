# Round-2 check 2: full GPU suite (no -x), smoke, cfg4 regression hunt (core SVD / rotation switches)
set -x
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/c4_default.log 2>&1
ADROM_CORE_JACOBI=1 timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/c4_jacobi.log 2>&1
ADROM_NO_TC_ROT=1 timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/c4_notc.log 2>&1
tail -n 3 gpurun_out/pytest_gpu2.log gpurun_out/smoke2.log

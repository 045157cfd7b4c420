set -x
(cd bisect/f25 && ADROM_CORE_JACOBI=1 timeout 600 python bench.py --config cfg4 --no-cpu-baseline > ../../gpurun_out/bisect_f25_jacobi.log 2>&1)
(cd bisect/hyb_linalg && timeout 600 python bench.py --config cfg4 --no-cpu-baseline --steps 200 --warmup 3 --no-e2e > ../../gpurun_out/bisect_hyb_long.log 2>&1)

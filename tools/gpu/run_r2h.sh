set -x
(cd bisect/head_oldcore && timeout 900 python tools/core_ab.py > ../../gpurun_out/core_ab.log 2>&1)
(cd bisect/head_oldcore && ADROM_CORE_JACOBI=1 timeout 900 python tools/core_ab.py > ../../gpurun_out/core_ab_jac.log 2>&1)
tail -n 6 gpurun_out/core_ab.log gpurun_out/core_ab_jac.log

set -x
(cd bisect/head_oldcore && ADROM_ROOT=$PWD timeout 900 python tools/core_ab_session.py new 5 > ../../gpurun_out/c4ab_new.log 2>&1; cp gpurun_out/c4ab_new.npz ../../gpurun_out/ 2>/dev/null)
(cd bisect/head_oldcore && ADROM_CORE_OLD=1 ADROM_ROOT=$PWD timeout 900 python tools/core_ab_session.py old 5 > ../../gpurun_out/c4ab_old.log 2>&1; cp gpurun_out/c4ab_old.npz ../../gpurun_out/ 2>/dev/null)
tail -n 8 gpurun_out/c4ab_new.log gpurun_out/c4ab_old.log

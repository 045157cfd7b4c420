set -x
timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect.log 2>&1
ADROM_FACTORED=0 timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_explicit.log 2>&1
cat gpurun_out/cfg3_defect.log gpurun_out/cfg3_defect_explicit.log | grep step

set -x
ADROM_DEFECT_N=65536 timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_2p16.log 2>&1
ADROM_DEFECT_N=65536 ADROM_FACTORED=1 timeout 900 python tools/cfg3_defect.py > gpurun_out/cfg3_defect_2p16_fact.log 2>&1
grep step gpurun_out/cfg3_defect_2p16.log gpurun_out/cfg3_defect_2p16_fact.log

# Round-2 check 5: cfg3 bad-step restarts; cfg4 hybrid bisection (f25eec0 with old linalg / old physics)
set -x
timeout 1500 python tools/cfg3_badstep_diag.py > gpurun_out/cfg3_badstep.log 2>&1
for h in hyb_linalg hyb_phys; do
  (cd bisect/$h && timeout 600 python bench.py --config cfg4 --no-cpu-baseline > ../../gpurun_out/bisect_$h.log 2>&1)
done
tail -n 5 gpurun_out/cfg3_badstep.log

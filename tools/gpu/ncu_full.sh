# usage: bash tools/gpu/ncu_full.sh <kernel-regex> <out-name> <count> -- bench args...
set -x
K="$1"; OUT="$2"; CNT="$3"; shift 4
export ADROM_PROFILE_TIMED=1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:$K" -c "$CNT" -o "gpurun_out/$OUT" python bench.py "$@" --no-cpu-baseline --no-e2e > "gpurun_out/$OUT.log" 2>&1
python tools/profile_summary.py full "gpurun_out/$OUT.ncu-rep" "gpurun_out/$OUT.txt" "$OUT"
cat "gpurun_out/$OUT.txt"

#!/bin/bash
# compute-sanitizer over every cross-CTA protocol (tools/sanitize_cases.py), one
# process per (tool, case) so the once-per-process env knobs of k3c_repair /
# k3c_cert take effect.  Logs: gpurun_out/sanitize/<tool>_<case>.log, summary
# in gpurun_out/sanitize/summary.txt.  Usage: tools/sanitize.sh [tools...]
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
TOOLS=${*:-memcheck racecheck synccheck initcheck}
CASES=$(python - <<'PY'
import re
src = open("tools/sanitize_cases.py").read()
print(" ".join(re.findall(r"^def case_(\w+)", src, re.M)))
PY
)
CS=/usr/local/cuda/bin/compute-sanitizer
export PYTORCH_NO_CUDA_MEMORY_CACHING=1   # every torch allocation is its own block: memcheck sees overruns
for tool in $TOOLS; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no --check-device-heap yes"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  [ "$tool" = initcheck ] && extra="--track-unused-memory no"
  for c in $CASES; do
    log=$OUT/${tool}_${c}.log
    timeout 900 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    errs=$(grep -m1 -E "ERROR SUMMARY|RACECHECK SUMMARY" $log)
    echo "$tool $c rc=$rc ${errs}" | tee -a $OUT/summary.txt
  done
done

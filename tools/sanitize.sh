#!/bin/bash
# compute-sanitizer over every kernel family (run under gpurun, one GPU).
# Summaries -> gpurun_out/${R}_sanitizer_<tool>_<case>.txt (last lines: error count).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${ROUND:-r02}
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in ${CASES:-map cir build edge}; do
    out=gpurun_out/${R}_sanitizer_${tool}_${c}.txt
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = initcheck ] && extra="--track-unused-memory no"
    timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 20 \
      python tools/sanitize_cases.py $c > $out.full 2>&1
    echo "rc=$?" >> $out.full
    (grep -E "^(========= (ERROR SUMMARY|LEAK SUMMARY|RACECHECK SUMMARY|Invalid|Program hit|Race|Barrier|Uninitialized|Leaked)|.* ok|rc=)" $out.full | head -40) > $out
    tail -3 $out.full >> $out
    rm -f $out.full
  done
done
echo sanitize done

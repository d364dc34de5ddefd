#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every tools/sanit.py case, on
# this library's kernels only; one log per tool and case in gpurun_out/sanitize/, summary lines in
# gpurun_out/sanitize/summary.txt.  Run under gpurun: bash tools/sanitize.sh [cases...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CASES=${*:-"cfg1 cfg2 cfg3 mixed staged idx binary fallback nosigma tp host"}
: > gpurun_out/sanitize/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    log=gpurun_out/sanitize/${tool}_${c}.log
    timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=qrita --print-limit 20 \
      python tools/sanit.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(grep -c '^ok' $log) ok" \
      >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt

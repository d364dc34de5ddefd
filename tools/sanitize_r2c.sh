#!/bin/bash
# Sanitizer pass over the row tail after the composite in-bin ranking (X's index half reused).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
: > gpurun_out/sanitize/summary_r2c.txt
run() {
  local tool=$1 c=$2
  local log=gpurun_out/sanitize/r2c_${tool}_${c}.log
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=qrita --print-limit 20 python tools/sanit.py $c > $log 2>&1
  echo "$tool $c rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(grep -c '^ok' $log) ok" >> gpurun_out/sanitize/summary_r2c.txt
}
for c in cfg2 mixed staged; do run racecheck $c; done
for c in cfg2 mixed staged idx; do run memcheck $c; done
cat gpurun_out/sanitize/summary_r2c.txt

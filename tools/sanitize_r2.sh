#!/bin/bash
# Round-2 sanitizer pass (bounded): the kernels changed or added this round on their main cases.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
: > gpurun_out/sanitize/summary_r2.txt
run() {
  local tool=$1 c=$2
  local log=gpurun_out/sanitize/r2_${tool}_${c}.log
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=qrita --print-limit 20 python tools/sanit.py $c > $log 2>&1
  echo "$tool $c rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(grep -c '^ok' $log) ok" >> gpurun_out/sanitize/summary_r2.txt
}
for c in cfg2 cfg3 mixed tp lmhead; do run racecheck $c; done
for c in cfg3 tp host lmhead; do run synccheck $c; done
for c in cfg3 tp idx host lmhead; do run memcheck $c; done
run initcheck cfg3
cat gpurun_out/sanitize/summary_r2.txt

set -u
mkdir -p gpurun_out/sanitize
: > gpurun_out/sanitize/summary_r2b.txt
run() {
  local tool=$1 c=$2
  local log=gpurun_out/sanitize/r2b_${tool}_${c}.log
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=qrita --print-limit 20 python tools/sanit.py $c > $log 2>&1
  echo "$tool $c rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(grep -c '^ok' $log) ok" >> gpurun_out/sanitize/summary_r2b.txt
}
for c in tp host hostsparse lmhead; do run memcheck $c; done
for c in tp host hostsparse; do run racecheck $c; done
run synccheck tp
cat gpurun_out/sanitize/summary_r2b.txt

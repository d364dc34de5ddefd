#!/bin/bash
# Round-2 evidence run (under gpurun): bench lines for every config, the reference arm, ncu launch
# lists and --set full captures.  Output: gpurun_out/r2/ (+ gpurun_out/prof/ from round_profile.sh).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
python bench.py --steps 50 --warmup 5 > gpurun_out/r2/bench_cfg2.json 2> gpurun_out/r2/bench_cfg2.err
for c in cfg1 cfg3 cfg4 cfg2copy; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
python bench.py --config cfg5 --steps 20 --warmup 5 > gpurun_out/r2/bench_cfg5.json 2> gpurun_out/r2/bench_cfg5.err
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r2/reference_cfg2.json 2> gpurun_out/r2/reference_cfg2.err
python bench.py --impl reference --config cfg4 --steps 3 --warmup 1 > gpurun_out/r2/reference_cfg4.json 2> gpurun_out/r2/reference_cfg4.err
python tools/e2e_pageable.py > gpurun_out/r2/e2e_pageable.txt 2>&1
python tools/diag.py ftiming cfg2 > gpurun_out/r2/ftiming_cfg2.txt 2>&1
python tools/diag.py t16timing > gpurun_out/r2/t16timing.txt 2>&1
bash tools/round_profile.sh
tail -c 400 gpurun_out/r2/*.json

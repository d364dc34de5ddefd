timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 120 python tools/diag.py ftiming cfg2 cfg4 cfg1 2>&1 | grep -v "0/" > gpurun_out/ftiming.log
for c in cfg2 cfg4 cfg1 cfg3 cfg2copy; do timeout 300 python bench.py --config $c --no-extras > gpurun_out/bench_$c.log 2>&1; done

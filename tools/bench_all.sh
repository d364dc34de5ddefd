# quick perf sweep: fused path on every config, plus the staged ablation on cfg2
for c in cfg2 cfg4 cfg1 cfg3 cfg2copy; do timeout 300 python bench.py --config $c --no-extras > gpurun_out/bench_$c.log 2>&1; done
timeout 200 python tools/graph_exp.py cfg2 > gpurun_out/graph.log 2>&1

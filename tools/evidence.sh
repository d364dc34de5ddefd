# full bench line (cfg2), reference arm, then ncu evidence
timeout 300 python bench.py > gpurun_out/bench_cfg2_full.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for c in cfg4 cfg3 cfg1 cfg2copy; do timeout 300 python bench.py --config $c --no-extras > gpurun_out/bench_$c.log 2>&1; done
bash tools/round_profile.sh

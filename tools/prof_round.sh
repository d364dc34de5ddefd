# round evidence: 3 bench repeats (variance), ncu launch list and one --set full capture of qrita_fused (cfg2)
for r in 1 2 3; do timeout 300 python bench.py --no-extras > gpurun_out/bench_rep$r.log 2>&1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 6 -c 6 --csv \
    --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qrita_fused -s 3 -c 1 \
    -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/prof_fused.log 2>&1
for c in cfg4 cfg3 cfg1; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qrita -s 3 -c 2 --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
done

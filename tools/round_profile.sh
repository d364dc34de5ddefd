# Round evidence (run under gpurun): ncu launch lists for every config and --set full captures of the
# dominant kernels (qrita_fused on cfg2, qrita_topp16 on cfg3).  Numbers printed under ncu are never
# bench values.  Summarise with: python tools/summarize_profiles.py <tag>
mkdir -p gpurun_out/prof
for c in cfg2 cfg4 cfg3 cfg1 cfg5 cfg2copy; do
  # cfg5: the TP kernels (qrita::tp::tp_*) next to the shard's qrita_fused
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k "regex:qrita|tp_" -s 3 -c 12 --csv --log-file gpurun_out/prof/launches_$c.csv \
      python bench.py --config $c --steps 3 --warmup 3 --no-extras > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:qrita_fused -s 3 -c 1 \
    -o gpurun_out/prof/fused_cfg2 python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/prof/fused_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qrita_topp16 -s 3 -c 1 \
    -o gpurun_out/prof/topp16_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-extras \
    > gpurun_out/prof/topp16_cfg3.log 2>&1
# LM-head fusion: launch list of the fused call and a full capture of lmh_gemm
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:lmh_gemm|qrita_tail" -c 6 --csv --log-file gpurun_out/prof/launches_lmhead.csv \
    python tools/lmh_prof.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lmh_gemm -s 1 -c 1 \
    -o gpurun_out/prof/lmhead_gemm python tools/lmh_prof.py > gpurun_out/prof/lmhead_gemm.log 2>&1

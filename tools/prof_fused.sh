# ncu full capture of the fused kernel on cfg2 with dense warp-state sampling (source-level stalls)
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --warp-sampling-buffer-size 268435456 -k regex:qrita_fused -s 3 -c 1 \
    -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/prof_fused.log 2>&1

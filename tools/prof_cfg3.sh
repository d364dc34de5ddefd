ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:qrita_fused -s 3 -c 1 \
    -o gpurun_out/prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-extras > gpurun_out/prof_cfg3.log 2>&1

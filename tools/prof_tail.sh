# one ncu --set full capture of the row tail on cfg2 (source-level stall reasons)
ncu --set full --clock-control none --import-source on -k regex:qrita_tail -s 3 -c 1 \
    -o gpurun_out/prof_tail python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/prof_tail.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qrita_stream -s 3 -c 1 \
    -o gpurun_out/prof_stream python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/prof_stream.log 2>&1

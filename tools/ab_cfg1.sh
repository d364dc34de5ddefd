# A/B of build/ab/a.so vs b.so on cfg1 (latency) and cfg2, interleaved.
rm -f gpurun_out/ab.txt
for v in a b a b a b; do
  for cfg in cfg1 cfg2; do
    QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 50 --config $cfg > gpurun_out/ab_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v $cfg', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt
  done
done

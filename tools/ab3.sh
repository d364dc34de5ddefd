# A/B/C of three builds (build/ab/{a,b,c}.so) on cfg2 and cfg3 (cfg4 once each), interleaved.
rm -f gpurun_out/ab.txt
for v in a b c a b c; do
  for cfg in cfg2 cfg3; do
    QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 30 --config $cfg > gpurun_out/ab_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v $cfg', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt
  done
done
for v in a b c; do
  QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 10 --config cfg4 > gpurun_out/ab4_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab4_$v.log').read().strip().splitlines()[-1]); print('$v cfg4', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt
done

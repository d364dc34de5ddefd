# A/B of two builds (build/ab/a.so vs build/ab/b.so) on cfg2 (masked), cfg2 index-only and cfg4, interleaved.
rm -f gpurun_out/ab.txt
for v in a b a b a b; do
  QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 30 > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v cfg2', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt
  QRITA_LIB=build/ab/$v.so FLUSH=1 IDX=1 timeout 100 python tools/diag.py ftiming cfg2 2>&1 | grep "last end" | sed "s/^/$v idx /" >> gpurun_out/ab.txt
  QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 10 --config cfg4 > gpurun_out/ab4_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab4_$v.log').read().strip().splitlines()[-1]); print('$v cfg4', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt
done

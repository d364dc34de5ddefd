for v in k2 l m k2 l m; do QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 30 > gpurun_out/ab_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt; done
for v in k2 l m; do QRITA_LIB=build/ab/$v.so timeout 120 python tools/diag.py smid cfg2 2>&1 | grep rep0 | sed "s/^/$v /" >> gpurun_out/ab.txt; done

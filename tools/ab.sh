for v in p q r p q r; do QRITA_LIB=build/ab/$v.so timeout 300 python bench.py --no-extras --steps 30 > gpurun_out/ab_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v cfg2', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt; done

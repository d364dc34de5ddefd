for v in 0 1 0 1 0 1; do if [ $v = 1 ]; then export QRITA_NO_SPREAD=1; else unset QRITA_NO_SPREAD; fi; timeout 300 python bench.py --no-extras --steps 30 > gpurun_out/ab_$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('nospread=$v', round(d['ms_per_step']*1e3,2))" >> gpurun_out/ab.txt; done
unset QRITA_NO_SPREAD; timeout 120 python tools/diag.py smid cfg2 2>&1 | grep rep0 >> gpurun_out/ab.txt

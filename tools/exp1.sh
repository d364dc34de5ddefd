for cta in 3 2; do for pub in 0 1; do
QRITA_STREAM_CTAS_PER_SM=$cta QRITA_EXP_PUBLISH=$pub python bench.py --no-extras --steps 30 > gpurun_out/exp_${cta}_${pub}.log 2>&1
done; done

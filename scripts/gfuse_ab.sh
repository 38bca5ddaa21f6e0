# A/B of the G-fused backward (NEXT-4b) against the materialised G: step and kernel times
for cfg in ${CFGS:-c2 c4}; do for g in 1 0; do for e in ${EPIS:-default}; do
  if [ "$e" = default ]; then unset WHALE_BWD_EPI; else export WHALE_BWD_EPI=$e; fi
  WHALE_GFUSE=$g python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_${cfg}_g$g.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_${cfg}_g$g.json').read().strip().splitlines()[-1]);print('$cfg gfuse=$g epi=$e', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done; done; done

# A/B of runtime knobs on one config: KNOBS="VAR=val VAR2=val ..." entries separated by ';'
CFG=${CFG:-c4}
IFS=';' read -ra SETS <<< "${KNOBS:-NONE=0}"
for set in "${SETS[@]}"; do
  env $set python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-autograd > gpurun_out/b_knob.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_knob.json').read().strip().splitlines()[-1]);print('$CFG [$set]', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/b_knob.json
done

# multi-GPU bench A/B of runtime knobs (run under gpurun --gpus N): KNOBS="A=1;A=0"
N=${N:-2}
IFS=';' read -ra SETS <<< "${KNOBS:-NONE=0}"
port=29600
for set in "${SETS[@]}"; do
  port=$((port+1))
  env $set python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/b_mg.json 2> gpurun_out/b_mg.err
  python -c "import json;d=json.loads(open('gpurun_out/b_mg.json').read().strip().splitlines()[-1]);print('N=$N [$set]', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/b_mg.err
done

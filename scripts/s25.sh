set -u
O=gpurun_out/s25; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
for M in 0 4 1 5 8 0 2; do
WHALE_PDL_MASK=$M timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$M bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline > $O/b.json 2> $O/b.err; 
python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('N=$N mask=$M', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})" || tail -3 $O/b.err
done
for M in 0 1 2 3 8 0; do
WHALE_PDL_MASK=$M CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-autograd > $O/b1.json 2> $O/b1.err
python -c "import json;d=json.loads(open('$O/b1.json').read().strip().splitlines()[-1]);print('N=1 mask=$M', round(d['ms_per_step']*1e3,1), round(d['value']))" || tail -3 $O/b1.err
done

# N=2 diagnostics: timeline, per-kernel times, bench
set -u
O=gpurun_out/s2; mkdir -p $O
for C in c2; do
CFG=$C timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/trace_step.py > $O/trace_${C}_n2.txt 2> $O/trace_${C}_n2.err; echo "trace rc=$?"
CFG=$C timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 scripts/mgpu_times.py > $O/times_${C}_n2.txt 2> $O/times_${C}_n2.err; echo "times rc=$?"
done
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 30 --warmup 5 > $O/bench_c2_n2.json 2> $O/bench_c2_n2.err; echo "bench rc=$?"
cat $O/trace_c2_n2.txt $O/times_c2_n2.txt
python -c "import json;d=json.loads(open('$O/bench_c2_n2.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d.get('kernels'))"
CFG=c2 timeout 300 python scripts/trace_step.py > $O/trace_c2_n1.txt 2>&1; cat $O/trace_c2_n1.txt

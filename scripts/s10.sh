set -u
O=gpurun_out/s10; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py tests/test_emulated_ranks.py -q -x > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pt.log
for F in 1 0; do
WHALE_FUSED_GATHER=$F timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2960$F bench.py --gpus 2 --steps 30 --warmup 5 > $O/bench_f$F.json 2> $O/bench_f$F.err; echo "bench F=$F rc=$?"
python -c "import json;d=json.loads(open('$O/bench_f$F.json').read().strip().splitlines()[-1]);print('F=$F', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
WHALE_FUSED_GATHER=$F timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2961$F scripts/trace_step.py > $O/trace_f$F.txt 2>&1; grep '"it": 4' $O/trace_f$F.txt
done

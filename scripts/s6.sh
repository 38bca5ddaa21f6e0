set -u
O=gpurun_out/s6; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f1 or c2_full or graph or random or forward_only" > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pt.log
WHALE_F1_DBG=1 timeout 120 python scripts/trace_step.py > $O/tr_graph.txt 2>&1; cat $O/tr_graph.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"

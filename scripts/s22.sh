set -u
O=gpurun_out/s22; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pt.log
timeout 300 python bench.py --steps 50 --warmup 5 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c2_n1.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1), d['value'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['roofline']['frac'], d['e2e']['value'], d['autograd'])"
for CF in c4 c5; do
timeout 300 python bench.py --config $CF --steps 10 --warmup 3 --no-cpu-baseline --no-autograd > $O/bench_$CF.json 2> $O/bench_$CF.err; echo "bench $CF rc=$?"
python -c "import json;d=json.loads(open('$O/bench_$CF.json').read().strip().splitlines()[-1]);print('$CF', round(d['ms_per_step']*1e3,1), d['value'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['roofline'], d['clocks'])"
done

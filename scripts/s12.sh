set -u
O=gpurun_out/s12; mkdir -p $O
cat gpurun_out/s11/*.txt > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bwd_cta_pairs" > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pt.log
for E in 2 4 6; do
WHALE_BWD_EPI=$E timeout 300 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --no-autograd > $O/c5_e$E.json 2> $O/c5_e$E.err; echo "c5 epi=$E rc=$?"
python -c "import json;d=json.loads(open('$O/c5_e$E.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'])"
done
WHALE_BWD_PAIR=0 timeout 300 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --no-autograd > $O/c5_np.json 2> $O/c5_np.err; echo "c5 nopair rc=$?"
python -c "import json;d=json.loads(open('$O/c5_np.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'])"

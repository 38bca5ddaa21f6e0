set -u
O=gpurun_out/s13; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pt.log
timeout 300 python bench.py --steps 50 --warmup 5 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_c2_n1.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1), d['value'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['roofline'])"
python scripts/run_steps.py --config c5 --steps 2 > $O/rs_c5.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"splitfc_gemm|splitfc_bwd" -s 2 -c 2 -o $O/prof_c5 python scripts/run_steps.py --config c5 --steps 2 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"

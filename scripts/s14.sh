set -u
O=gpurun_out/s14; mkdir -p $O
for r in 1 2; do
for L in old new; do
  if [ $L = old ]; then export WHALE_LIB_PATH=$PWD/paper_2011_09208_b200/lib/libwhale_splitfc_old.so; else unset WHALE_LIB_PATH; fi
  timeout 120 python scripts/trace_step.py > $O/t_$L.txt 2>&1; echo "$L $(tail -1 $O/t_$L.txt)"
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-autograd > $O/b_$L.json 2> $O/b_$L.err
  python -c "import json;d=json.loads(open('$O/b_$L.json').read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done
done
unset WHALE_LIB_PATH
timeout 300 python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline --no-autograd > $O/c5.json 2> $O/c5.err; echo "c5 rc=$?"
python -c "import json;d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'], d['roofline'])"

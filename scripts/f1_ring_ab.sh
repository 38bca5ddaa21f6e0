# F1 A/B: G1 (HBM) ring slots vs G2 (L2 re-read) ring slots, single vs split MMA issue, c2 N=1
for cfg in ${CFGS:-"8 2 0" "4 3 0" "3 4 0" "8 2 1" "4 3 1" "3 4 1"}; do
  set -- $cfg
  WHALE_F1_S1=$1 WHALE_F1_S2=$2 WHALE_F1_SPLIT=$3 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-autograd > gpurun_out/b_f1.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b_f1.json').read().strip().splitlines()[-1]);print('S1<=$1 S2=$2 split=$3', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done

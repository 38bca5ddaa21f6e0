set -u
O=gpurun_out/s18; mkdir -p $O
for PF in 0 4 8 16 24 32 0; do
  WHALE_F1_PF=$PF timeout 120 python scripts/trace_step.py > $O/t.txt 2>&1
  echo "PF=$PF $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
done

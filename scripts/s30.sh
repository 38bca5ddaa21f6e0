set -u
O=gpurun_out/s30; mkdir -p $O
for G in 0 1 0 1; do
  WHALE_GFUSE=$G CFG=c4 timeout 200 python scripts/trace_step.py > $O/t.txt 2>&1
  echo "c4 GFUSE=$G $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
done
for SH in "64 50000" "128 25000" "256 12500"; do
  set -- $SH
  for G in 0 1; do
  WHALE_GFUSE=$G B=$1 C=$2 timeout 200 python scripts/trace_step.py > $O/t.txt 2>&1
  echo "B=$1 C=$2 GFUSE=$G $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
  done
done

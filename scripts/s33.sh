set -u
O=gpurun_out/s33; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_emulated_ranks.py -q -x > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pt.log
for SH in "64 50000" "128 25000" "256 12500"; do
  set -- $SH
  for D in 1 0 1 0; do
  WHALE_P_DIRECT=$D B=$1 C=$2 timeout 200 python scripts/trace_step.py > $O/t.txt 2>&1
  echo "B=$1 C=$2 direct=$D $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
  done
done

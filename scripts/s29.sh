set -u
O=gpurun_out/s29; mkdir -p $O
for K in "WHALE_F1_G2K=128" "WHALE_F1_G2K=64 WHALE_F1_S2=4" "WHALE_F1_G2K=64 WHALE_F1_S2=5" "WHALE_F1_G2K=64 WHALE_F1_S2=6" "WHALE_F1_G2K=64 WHALE_F1_S2=3" "WHALE_F1_G2K=128"; do
  env $K timeout 120 python scripts/trace_step.py > $O/t.txt 2>&1
  echo "[$K] $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
done
WHALE_F1_G2K=64 WHALE_F1_S2=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f1 or c2_full or graph" > $O/pt.log 2>&1; echo "pytest g2k64 rc=$?"; tail -2 $O/pt.log

# backward store-path A/B at the N=2 / N=4 shard shapes and c4 (N = 1 emulation of one rank)
set -u
O=gpurun_out/s11; mkdir -p $O
for SH in "64 50000" "128 25000" "256 1000000"; do
  set -- $SH; B=$1; C=$2; D=2048; [ $B = 256 ] && D=512
  for K in "WHALE_BWD_EPI=2" "WHALE_BWD_EPI=4" "WHALE_BWD_EPI=6" "WHALE_ROW_BULK=2 WHALE_DW_BN=128" "WHALE_DW_BN=128"; do
    if [ $B = 256 ]; then CF=c4; else CF=c2; fi
    env $K CFG=$CF B=$B C=$C timeout 120 python scripts/trace_step.py > $O/t.txt 2>&1
    echo "B=$B C=$C [$K] $(tail -1 $O/t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["span_us"], d["win_us"])' 2>&1 | tail -1)"
  done
done

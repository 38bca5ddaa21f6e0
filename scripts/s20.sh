set -u
O=gpurun_out/s20; mkdir -p $O
for SH in "32 100000" "64 50000" "128 25000"; do
  set -- $SH
  BWD_TL=1 WHALE_EPI_DEBUG=16 B=$1 C=$2 timeout 120 python scripts/trace_step.py > $O/t_$1.txt 2>&1; echo "B=$1 C=$2"; tail -2 $O/t_$1.txt | cut -c1-250
done

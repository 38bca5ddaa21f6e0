set -u
O=gpurun_out/s21; mkdir -p $O
for SH in "32 100000" "64 50000" "128 25000"; do
  set -- $SH
  for K in 16 48; do
  BWD_TL=1 WHALE_EPI_DEBUG=$K B=$1 C=$2 timeout 120 python scripts/trace_step.py > $O/t_$1.txt 2>&1; echo "B=$1 C=$2 dbg=$K $(grep bwd_ctas $O/t_$1.txt | cut -c1-200)"; tail -1 $O/t_$1.txt | cut -c1-160
  done
done

set -u
O=gpurun_out/s23; mkdir -p $O
for r in 1 2; do
for L in old new; do
  if [ $L = old ]; then export WHALE_LIB_PATH=$PWD/paper_2011_09208_b200/lib/libwhale_splitfc_old.so; else unset WHALE_LIB_PATH; fi
  CFG=c5 ITERS=3 timeout 300 python scripts/trace_step.py > $O/t_$L.txt 2>&1; echo "$L $(tail -1 $O/t_$L.txt | cut -c1-150)"
done
done

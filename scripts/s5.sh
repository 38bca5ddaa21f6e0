set -u
O=gpurun_out/s5; mkdir -p $O
WHALE_F1_DBG=1 timeout 120 python scripts/trace_step.py > $O/tr_graph.txt 2>&1; cat $O/tr_graph.txt

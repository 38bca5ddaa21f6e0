set -u
O=gpurun_out/s8; mkdir -p $O
F1_CTA_DUMP=$O/cta.json WHALE_F1_DBG=65 timeout 120 python scripts/trace_step.py > $O/tr_graph.txt 2>&1; cat $O/tr_graph.txt

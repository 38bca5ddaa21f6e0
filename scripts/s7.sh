set -u
O=gpurun_out/s7; mkdir -p $O
F1_CTA_DUMP=$O/cta.json WHALE_F1_DBG=1 timeout 120 python scripts/trace_step.py > $O/tr_graph.txt 2>&1; cat $O/tr_graph.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pt.log
for B in 64 128; do C=$((3200000/B)); B=$B C=$C timeout 120 python scripts/trace_step.py > $O/tr_b$B.txt 2>&1; echo B=$B; tail -1 $O/tr_b$B.txt; WHALE_SHRINK_A=0 B=$B C=$C timeout 120 python scripts/trace_step.py > $O/tr_b${B}_old.txt 2>&1; tail -1 $O/tr_b${B}_old.txt; done

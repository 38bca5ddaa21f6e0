set -u
O=gpurun_out/s4; mkdir -p $O
WHALE_F1_DBG=1 timeout 120 python scripts/trace_step.py > $O/tr_graph.txt 2>&1; cat $O/tr_graph.txt
NOGRAPH=1 WHALE_F1_DBG=1 timeout 120 python scripts/trace_step.py > $O/tr_eager.txt 2>&1; cat $O/tr_eager.txt
B=64 C=50000 timeout 120 python scripts/trace_step.py > $O/tr_b64.txt 2>&1; cat $O/tr_b64.txt
B=128 C=25000 timeout 120 python scripts/trace_step.py > $O/tr_b128.txt 2>&1; cat $O/tr_b128.txt
python scripts/run_steps.py --B 64 --C 50000 --steps 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"splitfc_gemm|splitfc_bwd|stats" -s 3 -c 3 -o $O/prof_b64 python scripts/run_steps.py --B 64 --C 50000 --steps 3 > $O/ncu_b64.log 2>&1; echo "ncu rc=$?"

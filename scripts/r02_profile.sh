# Round-2 evidence run on one B200 (gpurun): bench lines, launch list, ncu captures.
# Writes gpurun_out/r02/*; the summaries that matter are copied into profiles/ by hand.
set -u
O=gpurun_out/r02
mkdir -p $O
# 1. bench lines (N = 1): c2 (the headline), c4, c5
python bench.py --steps 50 --warmup 5 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err; echo "bench c2 rc=$?"
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4_n1.json 2> $O/bench_c4_n1.err; echo "bench c4 rc=$?"
python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > $O/bench_c5_n1.json 2> $O/bench_c5_n1.err; echo "bench c5 rc=$?"
# 2. launch list of the c2 bench command (cold-cache, serialised: compare shares)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-autograd > $O/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2_n1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-autograd > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
# 3. full captures: c2 F1 + stats + backward (one step after warm-up), c5 logits + backward
python scripts/run_steps.py --config c2 --steps 3 > $O/rs_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"splitfc_fwd_dx|stats_grad|splitfc_bwd" -s 3 -c 3 \
    -o $O/prof_c2 python scripts/run_steps.py --config c2 --steps 3 > $O/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
python scripts/run_steps.py --config c5 --steps 2 > $O/rs_c5.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"splitfc_gemm|splitfc_bwd" -s 2 -c 2 \
    -o $O/prof_c5 python scripts/run_steps.py --config c5 --steps 2 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
# 4. G-fused backward A/B (NEXT-4b) and the autograd leg
CFGS="c2 c4 c5" EPIS=default bash scripts/gfuse_ab.sh > $O/gfuse_ab.txt 2>&1; echo "gfuse ab rc=$?"
python scripts/autograd_step.py > $O/autograd_c2.json 2>&1; echo "autograd rc=$?"

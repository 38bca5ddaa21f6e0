# Round-2 (second session) evidence run on one B200: bench lines (c2 / c4 / c5), the ncu launch
# list of the c2 bench command, ncu --set full captures of c2 (F1, stats, backward) and c5
# (paired logits + paired backward).  Writes gpurun_out/r02f/*; summaries are copied to profiles/.
set -u
O=gpurun_out/r02f; mkdir -p $O
python bench.py --steps 50 --warmup 5 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err; echo "bench c2 rc=$?"
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4_n1.json 2> $O/bench_c4_n1.err; echo "bench c4 rc=$?"
python bench.py --config c5 --steps 6 --warmup 3 --no-cpu-baseline > $O/bench_c5_n1.json 2> $O/bench_c5_n1.err; echo "bench c5 rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-autograd > $O/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2_n1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-autograd > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/run_steps.py --config c2 --steps 3 > $O/rs_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"splitfc_fwd_dx|stats_grad|splitfc_bwd" -s 3 -c 3 \
    -o $O/prof_c2 python scripts/run_steps.py --config c2 --steps 3 > $O/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
python scripts/run_steps.py --config c5 --steps 2 > $O/rs_c5.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"splitfc_gemm|splitfc_bwd" -s 2 -c 2 \
    -o $O/prof_c5 python scripts/run_steps.py --config c5 --steps 2 > $O/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
for f in $O/bench_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step']*1e3,1), d['value'], d['roofline']['frac'], d['clocks'])"; done

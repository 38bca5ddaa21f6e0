set -u
O=gpurun_out/s24; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29681 tests/mgpu_parity_worker.py > $O/mg.log 2>&1; echo "worker rc=$?"
python - <<PY
import json
rs=[json.loads(l) for l in open("$O/mg.log") if l.startswith("{")]
print(len(rs), "results; all ok:", all(r["ok"] for r in rs), "dx_rep:", all(r.get("dx_repeat_bitwise") for r in rs), "max dx_rel", max(r["dx_rel"] for r in rs))
PY
timeout 600 python -m pytest tests/test_emulated_ranks.py -q -x > $O/emu.log 2>&1; echo "emu rc=$?"; tail -1 $O/emu.log
for r in 1 2; do
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$((r+1)) bench.py --gpus $N --steps 30 --warmup 5 > $O/b.json 2> $O/b.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('N=$N', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done
CFG=c2 timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29685 scripts/trace_step.py > $O/trace.txt 2>&1; grep '"it": 4' $O/trace.txt | cut -c1-200

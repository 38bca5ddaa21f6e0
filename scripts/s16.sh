set -u
O=gpurun_out/s16; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
for RS in 1 0; do
WHALE_NVLS_RS=$RS timeout 900 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$RS tests/mgpu_parity_worker.py > $O/mg_rs$RS.log 2>&1; echo "worker RS=$RS rc=$?"
python - <<PY
import json
rs=[json.loads(l) for l in open("$O/mg_rs$RS.log") if l.startswith("{")]
print(len(rs), "results; all ok:", all(r["ok"] for r in rs), "nvls_rs:", {r.get("nvls_rs") for r in rs}, "dx_rep:", all(r.get("dx_repeat_bitwise") for r in rs), "max dx_rel", max(r["dx_rel"] for r in rs))
PY
WHALE_NVLS_RS=$RS timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2965$RS bench.py --gpus $N --steps 30 --warmup 5 > $O/b_rs$RS.json 2> $O/b_rs$RS.err; echo "bench RS=$RS rc=$?"
python -c "import json;d=json.loads(open('$O/b_rs$RS.json').read().strip().splitlines()[-1]);print('RS=$RS N=$N', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done

# Round-2 (second session) multi-GPU evidence on one 4-GPU box: parity worker at N = 4 and
# N = 2, bench lines c2 at N = 2 / 4 and c3 at N = 4, device timelines at N = 2 / 4.
set -u
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 tests/mgpu_parity_worker.py > $O/mgpu_parity_n4.log 2>&1; echo "worker n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 tests/mgpu_parity_worker.py > $O/mgpu_parity_n2.log 2>&1; echo "worker n2 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29703 bench.py --gpus 2 --steps 30 --warmup 5 > $O/bench_c2_n2.json 2> $O/bench_c2_n2.err; echo "bench c2 n2 rc=$?"
timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29704 bench.py --gpus 4 --steps 30 --warmup 5 > $O/bench_c2_n4.json 2> $O/bench_c2_n4.err; echo "bench c2 n4 rc=$?"
timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29705 bench.py --gpus 4 --config c3 --steps 30 --warmup 5 > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err; echo "bench c3 n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 CFG=c2 timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29706 scripts/trace_step.py > $O/timeline_c2_n2.txt 2>&1; echo "trace n2 rc=$?"
CFG=c2 timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29707 scripts/trace_step.py > $O/timeline_c2_n4.txt 2>&1; echo "trace n4 rc=$?"
for f in $O/bench_*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step']*1e3,1), round(d['value']), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'])"; done
for f in $O/mgpu_parity_n*.log; do python -c "
import json
rs=[json.loads(l) for l in open('$f') if l.startswith('{')]
print('$f', len(rs), 'ok', all(r['ok'] for r in rs), 'dx_rep', all(r.get('dx_repeat_bitwise') for r in rs))"; done

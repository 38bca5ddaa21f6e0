set -u
O=gpurun_out/s15; mkdir -p $O
for r in 1 2; do
for L in old new; do
  if [ $L = old ]; then export WHALE_LIB_PATH=$PWD/paper_2011_09208_b200/lib/libwhale_splitfc_old.so; else unset WHALE_LIB_PATH; fi
  CUDA_VISIBLE_DEVICES=0 timeout 120 python scripts/trace_step.py > $O/t_$L.txt 2>&1; echo "$L $(tail -1 $O/t_$L.txt | cut -c1-150)"
done
done
unset WHALE_LIB_PATH
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-autograd > $O/b.json 2> $O/b.err
python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('c2n1', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_emulated_ranks.py tests/test_gpu_parity.py -q -x -k "multigpu or emulated or f1 or pair or c2_full or graph" > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pt.log
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 30 --warmup 5 > $O/b2.json 2> $O/b2.err; echo "bench n2 rc=$?"
python -c "import json;d=json.loads(open('$O/b2.json').read().strip().splitlines()[-1]);print('c2n2', round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"

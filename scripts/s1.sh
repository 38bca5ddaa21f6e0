set -u
O=gpurun_out/s1; mkdir -p $O
nvidia-smi -L > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 > $O/bench_c2_n1.json 2> $O/bench_c2_n1.err; echo "bench rc=$?"
cat $O/bench_c2_n1.json | cut -c1-600

set -u
O=gpurun_out/s32; mkdir -p $O
python scripts/run_steps.py --B 128 --C 25000 --steps 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"splitfc_gemm" -s 2 -c 1 -o $O/prof_b128 python scripts/run_steps.py --B 128 --C 25000 --steps 3 > $O/ncu.log 2>&1; echo "ncu rc=$?"

set -u
O=gpurun_out/s3; mkdir -p $O
timeout 120 python scripts/f1_timeline.py > $O/f1_timeline.txt 2>&1; echo "tl rc=$?"
cat $O/f1_timeline.txt
export WHALE_LIB_PATH=$PWD/paper_2011_09208_b200/lib/libwhale_splitfc_timing.so
bash scripts/f1_modes.sh 2>&1 | tee $O/f1_modes.txt

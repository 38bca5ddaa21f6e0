set -u
O=gpurun_out/s17; mkdir -p $O
export WHALE_LIB_PATH=$PWD/paper_2011_09208_b200/lib/libwhale_splitfc_timing.so
bash scripts/f1_modes.sh 2>&1 | tee $O/f1_modes.txt

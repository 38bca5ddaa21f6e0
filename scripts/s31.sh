set -u
O=gpurun_out/s31; mkdir -p $O
timeout 900 python -m pytest tests/test_emulated_ranks.py -q -x -k "n8" > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pt.log

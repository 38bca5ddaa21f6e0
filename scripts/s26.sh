set -u
O=gpurun_out/s26; mkdir -p $O
timeout 900 python -m pytest tests/test_emulated_ranks.py -q -x -k "standalone_gather or bwd_cta_pairs" > $O/pt.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pt.log

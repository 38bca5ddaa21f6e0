#!/bin/bash
# F1 timing experiments: kernel time per WHALE_F1_DBG mode (2 = no G2, 4 = no epilogue, 8 = no G1 MMA)
for m in 0 2 6 14 4 12; do
  echo -n "mode $m: "
  WHALE_F1_DBG=$m timeout 120 python scripts/f1_probe.py 2>/dev/null | grep logits | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(round(d['logits_gemm']['total_ms']/d['logits_gemm']['launches']*1e3,1))"
done

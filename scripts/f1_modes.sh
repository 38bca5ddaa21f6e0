#!/bin/bash
# F1 timing experiments (timing-experiment build, WHALE_LIB_PATH): kernel time per WHALE_F1_DBG
# mode (2 = no G2, 4 = no epilogue, 8 = no G1 MMA); results other than the time are garbage.
for m in ${MODES:-0 2 4 6}; do
  echo -n "mode $m: "
  WHALE_F1_DBG=$m timeout 60 python scripts/f1_probe.py > /tmp/f1m.txt 2>&1
  tail -1 /tmp/f1m.txt | python -c "
import sys,json
try:
  d=json.loads(sys.stdin.read()); print(round(d['logits_gemm']['total_ms']/d['logits_gemm']['launches']*1e3,1))
except Exception as e: print('failed', open('/tmp/f1m.txt').read()[-300:])"
done

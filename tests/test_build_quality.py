"""The hot kernels compile without local-memory frames or register spills (-m "not gpu").

A dynamically indexed register array or a lambda capturing locals by reference makes ptxas
put them in local memory; in round 2 both happened unnoticed (F1 lost 6 us, the c4 logits
30 us).  The build log (`ptxas -v`, written by paper_2011_09208_b200/build.py) is checked
for every hot kernel instantiation."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "paper_2011_09208_b200", "lib", "ptxas.log")
HOT = ("splitfc_gemm_kernel", "splitfc_fwd_dx_kernel", "splitfc_bwd_kernel", "stats_grad_kernel",
       "stats_grad_multi_kernel", "bridge_gather_kernel")


def _entries():
    from paper_2011_09208_b200.build import build
    build()
    out, cur = {}, None
    for line in open(LOG):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            out[cur] = tuple(int(v) for v in m.groups())
    return out


def test_hot_kernels_have_no_local_memory():
    ents = _entries()
    hot = {k: v for k, v in ents.items() if any(h in k for h in HOT)}
    assert len(hot) >= 10, sorted(ents)  # every instantiation was found in the log
    bad = {k: v for k, v in hot.items() if any(v)}
    assert not bad, bad

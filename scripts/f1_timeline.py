"""F1 per-period timeline of CTA 0 at c2 (WHALE_F1_DBG=1): prints stamps relative to start (us)."""
import ctypes, os, sys
os.environ.setdefault("WHALE_F1_DBG", "1")
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE, _lib
L = _lib.lib()
B, C, D = 32, int(os.environ.get("C", 100000)), 2048
op = SplitFCSoftmaxCE(C, D, B)
X = syn.gen_features((0, B), D, 1, "bf16", device="cuda")
y = syn.gen_labels((0, B), C, 1, device="cuda").to(torch.int32)
W = syn.gen_weight((0, C), D, 1, "init", "bf16", device="cuda")
dx = torch.empty(B, D, dtype=torch.bfloat16, device="cuda"); dw = torch.empty(C, D, device="cuda")
for _ in range(4):
    op.forward(X, y, W); op.backward(W, dx, dw)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (1024 + 800))()
L.whale_debug_f1_timeline(buf)
t0 = min(buf[p * 16 + k] for p in range(64) for k in (0, 7) if buf[p * 16 + k])
names = ["mma_start", "g1_done", "mma_end", "epi_zfull", "epi_xfull", "epi_pfull", "epi_end", "prod_start",
         "e_maxbar", "e_refbar", "e_pempty", "e_ploop"]
print("period " + " ".join(n.rjust(9) for n in names))
for p in range(14):
    print(str(p).rjust(6), " ".join(("%9.2f" % ((buf[p * 16 + k] - t0) / 1e3)) if buf[p * 16 + k] else " " * 9 for k in range(12)))

ent = [buf[1024 + 5 * c] for c in range(148)]
st = [buf[1024 + 5 * c + 1] for c in range(148)]
en = [buf[1024 + 5 * c + 2] for c in range(148)]
g0 = min(st)
print("CTA entry: min %.2f max %.2f us rel. first post-prologue stamp; prologue max %.2f us" % (
    (min(ent) - g0) / 1e3, (max(ent) - g0) / 1e3, max((b - a) / 1e3 for a, b in zip(ent, st))))
import statistics
dur = [(e - s) / 1e3 for s, e in zip(st, en)]
print("CTA start spread us: %.2f  end: min %.2f median %.2f max %.2f (rel. first start)" % (
    (max(st) - g0) / 1e3, (min(en) - g0) / 1e3, statistics.median([(e - g0) / 1e3 for e in en]), (max(en) - g0) / 1e3))
slow = sorted(range(148), key=lambda c: -en[c])[:8]
print("slowest CTAs:", [(c, round((en[c] - g0) / 1e3, 1)) for c in slow])

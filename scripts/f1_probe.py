"""F1 probe: co-resident clusters and per-kernel times at c2 (N=1)."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE, _lib
L = _lib.lib()
cfg = syn.CONFIGS["c2"]
B = int(os.environ.get("B", cfg.B)); C = int(os.environ.get("C", cfg.C)); D = int(os.environ.get("D", cfg.D))
op = SplitFCSoftmaxCE(C, D, B)
c = op.config()
print(json.dumps({k: c[k] for k in ("f1", "f1_clusters", "f1_stages")}))
for smem in (150000, 200000, 222464):
    print("max_active_clusters(smem=%d) =" % smem, L.whale_debug_f1_max_clusters(smem))
X = syn.gen_features((0, B), D, 1, "bf16", device="cuda")
y = syn.gen_labels((0, B), C, 1, device="cuda").to(torch.int32)
W = syn.gen_weight((0, C), D, 1, "init", "bf16", device="cuda")
dx = torch.empty(B, D, dtype=torch.bfloat16, device="cuda"); dw = torch.empty(C, D, device="cuda")
for _ in range(3):
    op.forward(X, y, W); op.backward(W, dx, dw)
torch.cuda.synchronize()
op.profile(True)
for _ in range(20):
    op.forward(X, y, W); op.backward(W, dx, dw)
torch.cuda.synchronize()
print(json.dumps(op.profile_read()))

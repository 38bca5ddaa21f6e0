"""Small F1 + plain-path steps for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE
for (B, D, C) in [(32, 512, 1000), (17, 1024, 3001), (40, 192, 1000)]:
    X = syn.gen_features((0, B), D, 1, "bf16", device="cuda")
    y = syn.gen_labels((0, B), C, 1, device="cuda").to(torch.int32)
    W = syn.gen_weight((0, C), D, 1, "peaked", "bf16", device="cuda")
    b = syn.gen_bias((0, C), 1, 2.0, "bf16", device="cuda")
    op = SplitFCSoftmaxCE(C, D, B)
    for _ in range(2):
        op.forward(X, y, W, row_loss=True, bias=b, predictions=True)
        op.backward(W, bias_grad=True)
    op.check()
    torch.cuda.synchronize()
    print(B, D, C, "f1" if op.config()["f1"] else "plain", "ok", flush=True)

import sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle, synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE
B, D, C = 16, 64, 1000
for dt in ("f32", "bf16"):
    X = syn.gen_features((0, B), D, 1, dt); W = syn.gen_weight((0, C), D, 1, "init", dt); y = syn.gen_labels((0, B), C, 1)
    op = SplitFCSoftmaxCE(C, D, B, dtype=syn.torch_dtype(dt))
    cfg = op.config()
    wd = W.cuda(); loss = op.forward(X.cuda(), y.cuda(), wd)
    torch.cuda.synchronize()
    es = 4 if dt == "f32" else 2
    ldp = cfg["ldp"]
    ws = op.workspace
    P = ws[cfg["off_P"]:cfg["off_P"] + B * ldp * es].view(torch.float32 if es == 4 else torch.bfloat16).view(B, ldp)[:, :C].float().cpu().numpy()
    T = cfg["fwd"]["n_blocks"]; BN = cfg["fwd"]["BN"]
    mt = ws[cfg["off_m_tile"]:cfg["off_m_tile"] + B * T * 4].view(torch.float32).view(B, T).cpu().numpy()
    f = oracle.forward_backward(X, W, y.numpy())
    Z = f["Z"]
    Pref = np.exp(Z - np.repeat(mt, BN, axis=1)[:, :C])
    print(dt, "P err", np.abs(P - Pref).max(), "P sample", P[0, :4], Pref[0, :4])
    dx, dw = op.backward(wd); torch.cuda.synchronize()
    G = ws[cfg["off_P"]:cfg["off_P"] + B * ldp * es].view(torch.float32 if es == 4 else torch.bfloat16).view(B, ldp)[:, :C].float().cpu().numpy()
    print(dt, "G err", np.abs(G - f["G"]).max(), np.abs(f["G"]).max())
    part = ws[cfg["off_dxpart"]:cfg["off_dxpart"] + cfg["dx"]["splits"] * B * D * 4].view(torch.float32).view(-1, B, D).sum(0).cpu().numpy()
    print(dt, "dxpart err", np.abs(part - f["dX"]).max(), np.abs(f["dX"]).max(), "dx", dx.float().cpu().numpy()[0, :4], f["dX"][0, :4])
    print(dt, "dw", dw.cpu().numpy()[0, :4], f["dW"][0, :4], np.abs(dw.cpu().numpy() - f["dW"]).max())

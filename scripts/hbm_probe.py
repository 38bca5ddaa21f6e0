"""HBM read / write / copy bandwidth probe (torch kernels, CUDA events)."""
import json
import torch

n = 256 * 2 ** 20  # floats = 1 GiB
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
a.normal_()
res = {}


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


ms = t(lambda: b.fill_(1.0)); res["write_fill_GBps"] = n * 4 / ms / 1e6
ms = t(lambda: b.zero_()); res["write_zero_GBps"] = n * 4 / ms / 1e6
ms = t(lambda: b.copy_(a)); res["copy_rw_GBps"] = 2 * n * 4 / ms / 1e6
ms = t(lambda: a.sum()); res["read_sum_GBps"] = n * 4 / ms / 1e6
print(json.dumps(res))

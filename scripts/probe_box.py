"""Probe the GPU box: device properties, host cores, BLAS, symmetric memory support."""
import os, json, subprocess
import torch, numpy as np
out = {}
out["cuda"] = torch.cuda.is_available()
p = torch.cuda.get_device_properties(0)
out["name"] = p.name; out["sms"] = p.multi_processor_count; out["mem_gb"] = p.total_memory / 1e9
out["cc"] = [p.major, p.minor]
out["ndev"] = torch.cuda.device_count()
out["host_cores"] = len(os.sched_getaffinity(0))
import time
a = np.random.rand(2048, 2048); b = np.random.rand(2048, 2048)
t = time.time(); a @ b; out["np_fp64_gemm_gflops"] = 2 * 2048**3 / (time.time() - t) / 1e9
print(json.dumps(out))
print(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)

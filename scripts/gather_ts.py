"""Latency probe of the bridge gather (globaltimer stamps; WHALE_GATHER_DBG=16)."""
import ctypes, json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE, _lib
dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ["LOCAL_RANK"])); dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
cfg = syn.CONFIGS["c2"]
op = SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, group=dist.group.WORLD, device=dev)
X = syn.gen_features((rank * cfg.B, (rank + 1) * cfg.B), cfg.D, 1, device=dev)
y = syn.gen_labels((rank * cfg.B, (rank + 1) * cfg.B), cfg.C, 1, device=dev).to(torch.int32)
W = syn.gen_weight((op.o_r, op.o_r + op.C_r), cfg.D, 1, device=dev)
L = _lib.lib(); L.whale_debug_timestamps.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for it in range(6):
    op.forward(X, y, W); op.backward(W)
    buf = (ctypes.c_ulonglong * 32)()
    L.whale_debug_timestamps(buf, 32)
    t = list(buf)
    d0 = [t[i] - t[0] for i in range(6)]; d1 = [t[8 + i] - t[8] for i in range(6)]
    print(json.dumps({"rank": rank, "it": it, "blk0_ns": d0, "blkLast_ns": d1, "last_start_minus_first": t[8] - t[0]}), flush=True)
dist.barrier(); dist.destroy_process_group()

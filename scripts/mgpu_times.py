"""Per-kernel times at N>1 (torchrun): c2 shapes, library profiling hooks, no L2 flush."""
import json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE
dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
cfg = syn.CONFIGS[os.environ.get("CFG", "c2")]
seed = 1
op = SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, capacity=cfg.capacity, group=dist.group.WORLD, device=dev)
X = syn.gen_features((rank * cfg.B, (rank + 1) * cfg.B), cfg.D, seed, device=dev)
y = syn.gen_labels((rank * cfg.B, (rank + 1) * cfg.B), cfg.C, seed, device=dev).to(torch.int32)
W = syn.gen_weight((op.o_r, op.o_r + op.C_r), cfg.D, seed, device=dev)
dx = torch.empty(cfg.B, cfg.D, dtype=torch.bfloat16, device=dev); dw = torch.empty(op.C_r, cfg.D, device=dev)
def step():
    op.forward(X, y, W); op.backward(W, dx, dw)
for _ in range(5): step()
torch.cuda.synchronize(); dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): step()
b.record(); torch.cuda.synchronize()
t = a.elapsed_time(b) / 50 * 1e3
op.profile(True)
for _ in range(50): step()
k = op.profile_read(); op.check()
res = {"rank": rank, "tag": os.environ.get("TAG", ""), "step_us": round(t, 1),
       "k": {n: round(v["total_ms"] / v["launches"] * 1e3, 1) for n, v in k.items() if v["launches"]}}
out = [None] * world
dist.all_gather_object(out, res)
if rank == 0:
    for r in out: print(json.dumps(r))
dist.barrier(); dist.destroy_process_group()

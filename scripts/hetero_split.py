"""NEXT-1 experiment: hardware-aware uneven class split on emulated heterogeneous GPUs.

torchrun --nproc-per-node 2 scripts/hetero_split.py ; rank 1 is made a "half-speed GPU"
with WHALE_SM_LIMIT_R1=74 (its kernels use 74 of 148 SMs).  Times the c2 step (D=2048,
C=100K, B=32/GPU) for the even plan and for the capacity-proportional plan 2:1
("balances the FLOP ... through uneven sharding"), plus Alg. 1 with a memory
cap on rank 0.  Prints one JSON line per plan on rank 0.
"""
import json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local); dev = torch.device("cuda", local)
cfg = syn.CONFIGS["c2"]
res = []
# HETERO_CAP="2,2,1,1": capacity weights of the proportional plan (default 2:1:...:1)
capw = [int(v) for v in os.environ.get("HETERO_CAP", ",".join(["2"] + ["1"] * (world - 1))).split(",")]
tag = ":".join(str(v) for v in capw)
plans = [("even", None, None), (f"proportional {tag}", capw, None),
         (f"alg1 {tag}, rank0 capped at 55% of C", capw,
          [int(0.55 * cfg.C * cfg.D * 6)] + [10 ** 12] * (world - 1))]
for name, cap, mem in plans:
    op = SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, capacity=cap, group=dist.group.WORLD, device=dev, mem_bytes=mem)
    X = syn.gen_features((rank * cfg.B, (rank + 1) * cfg.B), cfg.D, 1, device=dev)
    y = syn.gen_labels((rank * cfg.B, (rank + 1) * cfg.B), cfg.C, 1, device=dev).to(torch.int32)
    W = syn.gen_weight((op.o_r, op.o_r + op.C_r), cfg.D, 1, device=dev)
    dx = torch.empty(cfg.B, cfg.D, dtype=torch.bfloat16, device=dev); dw = torch.empty(op.C_r, cfg.D, device=dev)
    def step():
        op.forward(X, y, W); op.backward(W, dx, dw)
    for _ in range(5): step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): step()
    g.replay(); torch.cuda.synchronize(); dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): g.replay()
    b.record(); torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 50 * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    op.check()
    res.append({"plan": name, "counts": op.counts, "step_us": round(float(t), 1),
                "samples_per_s": round(cfg.B * world / (float(t) / 1e6))})
    del op
if rank == 0:
    for r in res:
        caps = {k: v for k, v in os.environ.items() if k.startswith("WHALE_SM_LIMIT_R")}
        print(json.dumps({"world": world, "sm_limits": caps, **r}))
dist.barrier(); dist.destroy_process_group()

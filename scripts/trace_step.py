"""Device-side timeline of one split-FC step (kernel windows from the library tracer).

torchrun ... scripts/trace_step.py  (or plain python for N=1).  CFG env picks the config.
Graph-replays the step, arms the tracer, replays once, reads windows (ns rel. to step start).
"""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
from paper_2011_09208_b200 import SplitFCSoftmaxCE, _lib
world = int(os.environ.get("WORLD_SIZE", "1"))
group = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl")
    group = dist.group.WORLD
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local); dev = torch.device("cuda", local)
if os.environ.get("PERSIST_MB"):  # experiment: L2 set-aside for persisting (evict_last) lines
    torch.zeros(1, device=dev)
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
    rc = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(int(os.environ["PERSIST_MB"]) << 20))
    got = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(got), ctypes.c_int(0x06))
    print(json.dumps({"persisting_l2_set_rc": rc, "persisting_l2_bytes": got.value}))
cfg = syn.CONFIGS[os.environ.get("CFG", "c2")]
if os.environ.get("B") or os.environ.get("C"):  # shape overrides (e.g. one rank's shard shape at N = 1)
    import dataclasses
    cfg = dataclasses.replace(cfg, B=int(os.environ.get("B", cfg.B)), C=int(os.environ.get("C", cfg.C)))
op = SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, capacity=cfg.capacity, dtype=syn.torch_dtype(cfg.dtype), group=group, device=dev)
X = syn.gen_features((rank * cfg.B, (rank + 1) * cfg.B), cfg.D, 1, cfg.dtype, device=dev)
y = syn.gen_labels((rank * cfg.B, (rank + 1) * cfg.B), cfg.C, 1, device=dev).to(torch.int32)
W = syn.gen_weight((op.o_r, op.o_r + op.C_r), cfg.D, 1, "init", cfg.dtype, device=dev)
dx = torch.empty(cfg.B, cfg.D, dtype=syn.torch_dtype(cfg.dtype), device=dev)
dw = torch.empty(op.C_r, cfg.D, device=dev)
def step():
    op.forward(X, y, W); op.backward(W, dx, dw)
for _ in range(5): step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g): step()
g.replay(); torch.cuda.synchronize()
L = _lib.lib()
L.whale_debug_trace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
L.whale_debug_timestamps.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = ["gather", "logits", "stats", "grad", "dw", "dx", "rs_reduce", "transpose", "bwd", "bump"]
L.whale_debug_trace_enable(1)
out = []
for it in range(int(os.environ.get("ITERS", "5"))):
    if group is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if os.environ.get("NOGRAPH"):
        step()
    else:
        g.replay()
    buf = (ctypes.c_ulonglong * 32)()
    L.whale_debug_trace_read(buf)
    st = (ctypes.c_ulonglong * 32)()
    L.whale_debug_timestamps(st, 32)
    t0 = min(buf[2 * k] for k in range(16) if buf[2 * k + 1])
    rec = {names[k]: [round((buf[2 * k] - t0) / 1e3, 1), round((buf[2 * k + 1] - t0) / 1e3, 1)]
           for k in range(len(names)) if buf[2 * k + 1]}
    tend = max(v[1] for v in rec.values())
    stamps = {"row0": [round((st[16 + j] - t0) / 1e3, 1) for j in range(5) if st[16 + j] >= t0],
              "rowLast": [round((st[24 + j] - t0) / 1e3, 1) for j in range(5) if st[24 + j] >= t0],
              "rowLast_lastchunk": [round((st[21 + j] - t0) / 1e3, 1) for j in range(2) if st[21 + j] >= t0]}
    out.append({"rank": rank, "it": it, "span_us": tend, "win_us": rec, "stats_stamps": stamps})
L.whale_debug_trace_enable(0)
if os.environ.get("WHALE_F1_DBG"):  # F1 per-CTA [entry, after prologue, end] of the last replay
    tl = (ctypes.c_ulonglong * (1024 + 800))()
    L.whale_debug_f1_timeline(tl)
    ent = [tl[1024 + 5 * c] for c in range(148)]
    en = [tl[1024 + 5 * c + 2] for c in range(148)]
    cs = [tl[1024 + 5 * c + 3] for c in range(148)]
    ex = [tl[1024 + 5 * c + 4] for c in range(148)]
    span = lambda v: [round((min(v) - t0) / 1e3, 1), round((max(v) - t0) / 1e3, 1)]
    if all(ent):
        print(json.dumps({"rank": rank, "f1_cta_entry_us": span(ent), "f1_cta_end_us": span(en),
                          "f1_after_cluster_sync_us": span(cs), "f1_t0_at_exit_sync_us": span(ex)}))
        if os.environ.get("F1_CTA_DUMP"):
            rel = lambda v: [round((x - t0) / 1e3, 2) for x in v]
            json.dump({"entry": rel(ent), "end": rel(en), "sync": rel(cs), "exit": rel(ex)}, open(os.environ["F1_CTA_DUMP"], "w"))
if os.environ.get("GEMM_TL"):  # logits per-CTA timeline (needs WHALE_EPI_DEBUG=16)
    L.whale_debug_gemm_timeline.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    tg = (ctypes.c_ulonglong * 960)()
    L.whale_debug_gemm_timeline(tg)
    n = sum(1 for c in range(160) if tg[6 * c] and tg[6 * c + 5])
    cols = [[tg[6 * c + k] for c in range(160) if tg[6 * c] and tg[6 * c + 5]] for k in range(6)]
    g0 = min(cols[0])
    q = lambda v: [round((x - g0) / 1e3, 1) for x in (min(v), sorted(v)[len(v) // 2], max(v))]
    print(json.dumps({"rank": rank, "gemm_ctas": n, "entry": q(cols[0]), "after_prologue": q(cols[1]),
                      "last_load_issued": q(cols[2]), "last_mma_commit": q(cols[3]), "first_acc": q(cols[4]),
                      "epilogue_done": q(cols[5])}))
if os.environ.get("BWD_TL"):  # backward per-CTA timeline (needs WHALE_EPI_DEBUG=16)
    L.whale_debug_bwd_timeline.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    tb = (ctypes.c_ulonglong * 640)()
    L.whale_debug_bwd_timeline(tb)
    n = sum(1 for c in range(160) if tb[4 * c])
    st = [tb[4 * c] for c in range(n)]
    dxd = [tb[4 * c + 1] for c in range(n) if tb[4 * c + 1]]
    en = [tb[4 * c + 2] for c in range(n)]
    units = [tb[4 * c + 3] for c in range(n)]
    b0 = min(st)
    q = lambda v: [round((x - b0) / 1e3, 1) for x in (min(v), sorted(v)[len(v) // 2], max(v))] if v else []
    print(json.dumps({"rank": rank, "bwd_ctas": n, "start_min_med_max": q(st), "dx_done": q(dxd),
                      "end": q(en), "units_min_max": [min(units), max(units)]}))
op.check()
if group is not None:
    allo = [None] * world
    dist.all_gather_object(allo, out)
    if rank == 0:
        for o in allo:
            for r in o[-2:]:
                print(json.dumps(r))
    dist.barrier(); dist.destroy_process_group()
else:
    for r in out[-2:]:
        print(json.dumps(r))

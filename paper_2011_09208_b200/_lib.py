"""ctypes binding of include/whale_splitfc.h -- argument marshalling only.

Every step of the split-FC path runs inside libwhale_splitfc.so (hand-written sm_100a
CUDA).  There is no Python or CPU fallback: if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# WHALE_LIB_PATH: an alternative build of the same library (timing-experiment builds, scripts/ only)
LIB_PATH = os.environ.get("WHALE_LIB_PATH") or os.path.join(_HERE, "lib", "libwhale_splitfc.so")

STATUS = {
    0: "WHALE_OK", 1: "WHALE_ERR_INVALID_ARG", 2: "WHALE_ERR_UNSPLITTABLE", 3: "WHALE_ERR_UNSUPPORTED",
    4: "WHALE_ERR_STATE", 5: "WHALE_ERR_LABEL", 6: "WHALE_ERR_CUDA", 7: "WHALE_ERR_COMM",
}
WHALE_BF16, WHALE_F32 = 0, 1

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "whale_splitfc_plan", "whale_splitfc_plan_mem", "whale_splitfc_workspace_size", "whale_splitfc_create", "whale_splitfc_forward",
    "whale_splitfc_backward", "whale_splitfc_check", "whale_splitfc_destroy", "whale_last_error",
    "whale_splitfc_launches_per_step", "whale_splitfc_profile_enable", "whale_splitfc_profile_read",
    "whale_splitfc_config", "whale_splitfc_forward_ex", "whale_splitfc_backward_ex", "whale_splitfc_backward_scaled",
)


class WhaleError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world_size", ctypes.c_int32),
        ("local_batch", ctypes.c_int64),
        ("feature_dim", ctypes.c_int64),
        ("num_classes", ctypes.c_int64),
        ("shard_counts", ctypes.POINTER(ctypes.c_int64)),
        ("shard_offsets", ctypes.POINTER(ctypes.c_int64)),
        ("x_dtype", ctypes.c_int),
        ("dw_dtype", ctypes.c_int),
        ("peer_symm_ptrs", ctypes.POINTER(ctypes.c_void_p)),
        ("symm_bytes", ctypes.c_size_t),
        ("local_workspace", ctypes.c_void_p),
        ("local_workspace_bytes", ctypes.c_size_t),
        ("batch_counts", ctypes.POINTER(ctypes.c_int64)),
        ("multicast_ptr", ctypes.c_void_p),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libwhale_splitfc.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    st = ctypes.c_int
    vp = ctypes.c_void_p
    L.whale_splitfc_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint32),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    L.whale_splitfc_plan.restype = st
    L.whale_splitfc_plan_mem.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint32),
                                         ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    L.whale_splitfc_plan_mem.restype = st
    L.whale_splitfc_workspace_size.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(ctypes.c_size_t),
                                               ctypes.POINTER(ctypes.c_size_t)]
    L.whale_splitfc_workspace_size.restype = st
    L.whale_splitfc_create.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(vp)]
    L.whale_splitfc_create.restype = st
    L.whale_splitfc_forward.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.whale_splitfc_forward.restype = st
    L.whale_splitfc_backward.argtypes = [vp, vp, vp, vp, vp]
    L.whale_splitfc_backward.restype = st
    L.whale_splitfc_forward_ex.argtypes = [vp] * 10
    L.whale_splitfc_forward_ex.restype = st
    L.whale_splitfc_backward_ex.argtypes = [vp] * 6
    L.whale_splitfc_backward_ex.restype = st
    L.whale_splitfc_backward_scaled.argtypes = [vp] * 7
    L.whale_splitfc_backward_scaled.restype = st
    L.whale_splitfc_check.argtypes = [vp, vp]
    L.whale_splitfc_check.restype = st
    L.whale_splitfc_destroy.argtypes = [vp]
    L.whale_splitfc_destroy.restype = st
    L.whale_last_error.argtypes = []
    L.whale_last_error.restype = ctypes.c_char_p
    L.whale_splitfc_launches_per_step.argtypes = [vp]
    L.whale_splitfc_launches_per_step.restype = ctypes.c_int32
    L.whale_splitfc_profile_enable.argtypes = [vp, ctypes.c_int32]
    L.whale_splitfc_profile_enable.restype = st
    L.whale_splitfc_profile_read.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_int32)]
    L.whale_splitfc_profile_read.restype = st
    L.whale_splitfc_config.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.whale_splitfc_config.restype = st
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        raise WhaleError(status, where, lib().whale_last_error().decode())


def whale_splitfc_plan(num_classes: int, world_size: int, capacity=None):
    """-> (counts, offsets) lists; raises WhaleError on the C status."""
    L = lib()
    n = max(int(world_size), 1)
    counts = (ctypes.c_int64 * n)()
    offs = (ctypes.c_int64 * n)()
    cap = None
    if capacity is not None:
        if len(capacity) != int(world_size):
            raise ValueError(f"capacity has {len(capacity)} entries, world_size is {world_size}")
        cap = (ctypes.c_uint32 * len(capacity))(*[int(v) for v in capacity])
    _check(L.whale_splitfc_plan(int(num_classes), int(world_size), cap, counts, offs), "whale_splitfc_plan")
    return list(counts), list(offs)


def whale_splitfc_plan_mem(num_classes: int, world_size: int, capacity=None, mem_bytes=None,
                           bytes_per_class: int = 1, fixed_bytes: int = 0):
    """Algorithm 1 plan under memory caps -> (counts, offsets); raises WhaleError."""
    L = lib()
    n = max(int(world_size), 1)
    counts = (ctypes.c_int64 * n)()
    offs = (ctypes.c_int64 * n)()
    for name, v in (("capacity", capacity), ("mem_bytes", mem_bytes)):
        if v is not None and len(v) != int(world_size):
            raise ValueError(f"{name} has {len(v)} entries, world_size is {world_size}")
    cap = None if capacity is None else (ctypes.c_uint32 * len(capacity))(*[int(v) for v in capacity])
    mem = None if mem_bytes is None else (ctypes.c_uint64 * len(mem_bytes))(*[int(v) for v in mem_bytes])
    _check(L.whale_splitfc_plan_mem(int(num_classes), int(world_size), cap, mem, int(bytes_per_class),
                                    int(fixed_bytes), counts, offs), "whale_splitfc_plan_mem")
    return list(counts), list(offs)


def make_desc(rank, world, B, D, C, counts, offsets, x_dtype=WHALE_BF16, peer_ptrs=None, symm_bytes=0,
              workspace_ptr=0, workspace_bytes=0, batch_counts=None, dw_dtype=WHALE_F32, multicast_ptr=0):
    """Build a Desc; the returned tuple keeps the ctypes arrays alive.  batch_counts: optional
    per-rank DP batch [world] (NEXT-3); B must then be batch_counts[rank]."""
    c_counts = (ctypes.c_int64 * world)(*counts)
    c_offs = (ctypes.c_int64 * world)(*offsets)
    c_peers = None
    if peer_ptrs is not None:
        c_peers = (ctypes.c_void_p * world)(*peer_ptrs)
    c_batch = (ctypes.c_int64 * world)(*batch_counts) if batch_counts is not None else None
    d = Desc(rank, world, B, D, C, c_counts, c_offs, x_dtype, dw_dtype,
             ctypes.cast(c_peers, ctypes.POINTER(ctypes.c_void_p)) if c_peers is not None else None,
             symm_bytes, workspace_ptr or None, workspace_bytes, c_batch, multicast_ptr or None)
    return d, (c_counts, c_offs, c_peers, c_batch)


def whale_splitfc_workspace_size(desc: Desc):
    s, l_ = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib().whale_splitfc_workspace_size(ctypes.byref(desc), ctypes.byref(s), ctypes.byref(l_)),
           "whale_splitfc_workspace_size")
    return s.value, l_.value


def whale_splitfc_create(desc: Desc) -> int:
    h = ctypes.c_void_p()
    _check(lib().whale_splitfc_create(ctypes.byref(desc), ctypes.byref(h)), "whale_splitfc_create")
    return h.value


def whale_splitfc_forward(ctx, x_local, labels_local, w_shard, loss, row_loss, stream):
    _check(lib().whale_splitfc_forward(ctx, x_local, labels_local, w_shard, loss, row_loss or None, stream or None),
           "whale_splitfc_forward")


def whale_splitfc_backward(ctx, w_shard, dx_local, dw_shard, stream):
    _check(lib().whale_splitfc_backward(ctx, w_shard, dx_local, dw_shard, stream or None), "whale_splitfc_backward")


def whale_splitfc_forward_ex(ctx, x_local, labels_local, w_shard, bias, loss, row_loss, pred, prob, stream):
    _check(lib().whale_splitfc_forward_ex(ctx, x_local, labels_local, w_shard, bias or None, loss, row_loss or None,
                                          pred or None, prob or None, stream or None), "whale_splitfc_forward_ex")


def whale_splitfc_backward_ex(ctx, w_shard, dx_local, dw_shard, db_shard, stream):
    _check(lib().whale_splitfc_backward_ex(ctx, w_shard, dx_local, dw_shard, db_shard or None, stream or None),
           "whale_splitfc_backward_ex")


def whale_splitfc_backward_scaled(ctx, w_shard, dx_local, dw_shard, db_shard, grad_scale, stream):
    _check(lib().whale_splitfc_backward_scaled(ctx, w_shard, dx_local, dw_shard, db_shard or None, grad_scale or None,
                                               stream or None), "whale_splitfc_backward_scaled")


def whale_splitfc_check(ctx, stream):
    _check(lib().whale_splitfc_check(ctx, stream or None), "whale_splitfc_check")


def whale_splitfc_destroy(ctx):
    _check(lib().whale_splitfc_destroy(ctx), "whale_splitfc_destroy")


def whale_splitfc_launches_per_step(ctx) -> int:
    return int(lib().whale_splitfc_launches_per_step(ctx))


def whale_splitfc_profile_enable(ctx, enable: bool):
    _check(lib().whale_splitfc_profile_enable(ctx, 1 if enable else 0), "whale_splitfc_profile_enable")


def whale_splitfc_profile_read(ctx) -> dict:
    names = ctypes.create_string_buffer(1024)
    ms = (ctypes.c_double * 16)()
    n = (ctypes.c_int64 * 16)()
    k = ctypes.c_int32(0)
    _check(lib().whale_splitfc_profile_read(ctx, names, 1024, ms, n, 16, ctypes.byref(k)), "whale_splitfc_profile_read")
    out = {}
    for i, nm in enumerate(names.value.decode().split(";")[: k.value]):
        out[nm] = {"total_ms": ms[i], "launches": int(n[i])}
    return out


def whale_splitfc_config(ctx) -> dict:
    buf = ctypes.create_string_buffer(4096)
    _check(lib().whale_splitfc_config(ctx, buf, 4096), "whale_splitfc_config")
    return json.loads(buf.value.decode())

"""User-facing split-FC softmax cross-entropy (Whale hybrid strategy).

``SplitFCSoftmaxCE`` owns the device workspaces (torch allocations -- plumbing only) and a
context of libwhale_splitfc.so; ``forward``/``backward`` are the C-ABI calls on the current
torch stream.  For world > 1 the symmetric (peer-mapped) buffer comes from
``torch.distributed._symmetric_memory`` and all exchanges run in the library's own NVLink
kernels; the process group is used only for the rendezvous and a barrier.

``emulated_ranks`` builds N ranks on ONE device (the single-GPU test harness): the
"symmetric" buffers are plain allocations every rank's context addresses directly, so the
library's exchange kernels (bridge gather, statistics records, dX reduce-scatter) run
unchanged, each rank on its own stream.
"""
from __future__ import annotations

import os
from contextlib import contextmanager

import torch

from . import _lib


class SplitFCSoftmaxCE:
    """Class-split FC + softmax-CE over ``world`` ranks (shard r <-> rank r).

    Args:
        num_classes: C.  feature_dim: D.  local_batch: B (per rank; ignored if batch_counts).
        capacity: optional integer capacity weights (hardware-aware uneven class split).
        batch_counts: optional per-rank DP batch [world] (hardware-aware ``replicate``, NEXT-3;
            e.g. ``whale_splitfc_plan(B_tot, world, capacity)``); rank r's rows follow ranks < r.
        dtype: torch.bfloat16 (tcgen05 kind::f16) or torch.float32 (kind::tf32).
        dw_dtype: dtype of the dW_r the backward writes: torch.float32 (default) or, with bf16
            operands, torch.bfloat16 (fp32 accumulation, one rounding at the store) -- what a bf16
            weight's .grad wants, with no conversion pass.
        group: torch.distributed process group (None -> world 1).
    """

    def __init__(self, num_classes: int, feature_dim: int, local_batch: int, capacity=None,
                 dtype=torch.bfloat16, group=None, device=None, mem_bytes=None, bytes_per_class=None,
                 batch_counts=None, emulated=None, dw_dtype=torch.float32):
        self.C, self.D, self.B = int(num_classes), int(feature_dim), int(local_batch)
        self.dtype = dtype
        self.dw_dtype = dw_dtype
        dwdt = {torch.float32: _lib.WHALE_F32, torch.bfloat16: _lib.WHALE_BF16}[dw_dtype]
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if emulated is not None:  # (rank, world, [world] uint8 device buffers): see emulated_ranks
            self.rank, self.world = int(emulated[0]), int(emulated[1])
        elif group is not None:
            import torch.distributed as dist
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.group = group
        self.batch_counts = None
        if batch_counts is not None:
            self.batch_counts = [int(b) for b in batch_counts]
            if len(self.batch_counts) != self.world:
                raise ValueError("batch_counts must have one entry per rank")
            self.B = self.batch_counts[self.rank]
        self.row0 = sum(self.batch_counts[:self.rank]) if self.batch_counts else self.rank * self.B
        if mem_bytes is None:
            self.counts, self.offsets = _lib.whale_splitfc_plan(self.C, self.world, capacity)
        else:
            # Algorithm 1 under per-device memory caps (default cost: a W row in the operand
            # dtype + an fp32 dW row per class)
            es = 2 if dtype == torch.bfloat16 else 4
            bpc = bytes_per_class or self.D * (es + 4)
            self.counts, self.offsets = _lib.whale_splitfc_plan_mem(self.C, self.world, capacity, mem_bytes, bpc)
        self.C_r, self.o_r = self.counts[self.rank], self.offsets[self.rank]
        xdt = {torch.bfloat16: _lib.WHALE_BF16, torch.float32: _lib.WHALE_F32}[dtype]
        q, _keep = _lib.make_desc(self.rank, self.world, self.B, self.D, self.C, self.counts, self.offsets, xdt,
                                  batch_counts=self.batch_counts, dw_dtype=dwdt)
        symm_bytes, local_bytes = _lib.whale_splitfc_workspace_size(q)
        self.workspace = torch.empty(local_bytes, dtype=torch.uint8, device=self.device)
        peer_ptrs = None
        mc_ptr = 0
        self._symm = None
        if emulated is not None and self.world > 1:
            bufs = emulated[2]
            if len(bufs) != self.world or any(b.numel() < symm_bytes for b in bufs):
                raise ValueError(f"emulated ranks need {self.world} buffers of >= {symm_bytes} bytes")
            peer_ptrs = [int(b.data_ptr()) for b in bufs]
            self._symm = bufs
        elif self.world > 1:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(symm_bytes, dtype=torch.uint8, device=self.device)
            hdl = symm_mem.rendezvous(buf, group=group)
            buf.zero_()
            torch.cuda.synchronize(self.device)
            dist.barrier(group=group)
            peer_ptrs = [int(p) for p in hdl.buffer_ptrs]
            self._symm = (buf, hdl)
            # NVLS multicast address of the symmetric buffer when the NVSwitch supports it
            # (WHALE_NVLS=0 keeps the unicast all-gather)
            try:
                if os.environ.get("WHALE_NVLS", "1") != "0" and symm_mem._SymmetricMemory.has_multicast_support(
                        torch._C._autograd.DeviceType.CUDA, self.device.index):
                    mc_ptr = int(hdl.multicast_ptr or 0)
            except Exception:
                mc_ptr = 0
        self._desc, self._keep = _lib.make_desc(
            self.rank, self.world, self.B, self.D, self.C, self.counts, self.offsets, xdt, peer_ptrs, symm_bytes,
            self.workspace.data_ptr(), local_bytes, self.batch_counts, dwdt, mc_ptr)
        self.nvls = bool(mc_ptr)
        self.ctx = _lib.whale_splitfc_create(self._desc)
        self.loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.row_loss = torch.zeros(self.B, dtype=torch.float32, device=self.device)
        self.pred = torch.zeros(self.B, dtype=torch.int32, device=self.device)
        self.prob = torch.zeros(self.B, dtype=torch.float32, device=self.device)

    # ------------------------------------------------------------------ C-ABI calls
    def forward(self, x_local: torch.Tensor, labels_local: torch.Tensor, w_shard: torch.Tensor,
                row_loss: bool = False, bias: torch.Tensor | None = None, predictions: bool = False,
                loss_out: torch.Tensor | None = None):
        """-> device scalar loss (mean over the global batch).  labels: int32 (int64 is cast).

        bias: optional [C_r] FC bias shard (same dtype as W).  predictions=True also fills
        self.pred [B] (top-1 class over all C classes) and self.prob [B] (its probability).
        loss_out: optional fp32 scalar tensor the loss is written to (default: self.loss, reused
        by every call).
        """
        self._check_inputs(x_local, w_shard)
        if labels_local.dtype != torch.int32:
            labels_local = labels_local.to(torch.int32)
        self._labels = labels_local.contiguous()  # keep alive until the kernels ran
        self._x = x_local  # world 1: the backward reads x_local in place (header contract)
        if bias is not None and (bias.shape != (self.C_r,) or bias.dtype != self.dtype or not bias.is_contiguous()):
            raise ValueError(f"bias must be contiguous {self.dtype} [{self.C_r}]")
        stream = torch.cuda.current_stream(self.device).cuda_stream
        loss = self.loss if loss_out is None else loss_out
        if loss.dtype != torch.float32 or loss.numel() != 1 or loss.device != self.device:
            raise ValueError("loss_out must be a one-element fp32 tensor on the op's device")
        _lib.whale_splitfc_forward_ex(self.ctx, x_local.data_ptr(), self._labels.data_ptr(), w_shard.data_ptr(),
                                      bias.data_ptr() if bias is not None else None, loss.data_ptr(),
                                      self.row_loss.data_ptr() if row_loss else None,
                                      self.pred.data_ptr() if predictions else None,
                                      self.prob.data_ptr() if predictions else None, stream)
        return loss

    def backward(self, w_shard: torch.Tensor, dx_local: torch.Tensor | None = None,
                 dw_shard: torch.Tensor | None = None, db_shard: torch.Tensor | None = None, bias_grad: bool = False,
                 grad_scale: torch.Tensor | None = None):
        """-> (dX_r [B x D] in the operand dtype, dW_r [C_r x D] in dw_dtype[, db_r [C_r] fp32 if bias_grad]).

        grad_scale: optional device fp32 scalar g (d total / d loss): every output is multiplied
        by g inside the kernels that write it (whale_splitfc_backward_scaled)."""
        if dx_local is None:
            dx_local = torch.empty(self.B, self.D, dtype=self.dtype, device=self.device)
        if dw_shard is None:
            dw_shard = torch.empty(self.C_r, self.D, dtype=self.dw_dtype, device=self.device)
        if bias_grad and db_shard is None:
            db_shard = torch.empty(self.C_r, dtype=torch.float32, device=self.device)
        if grad_scale is not None and (grad_scale.dtype != torch.float32 or grad_scale.numel() != 1
                                       or grad_scale.device != self.device):
            raise ValueError("grad_scale must be a one-element fp32 tensor on the op's device")
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.whale_splitfc_backward_scaled(self.ctx, w_shard.data_ptr(), dx_local.data_ptr(), dw_shard.data_ptr(),
                                           db_shard.data_ptr() if db_shard is not None else None,
                                           grad_scale.data_ptr() if grad_scale is not None else None, stream)
        if db_shard is not None:
            return dx_local, dw_shard, db_shard
        return dx_local, dw_shard

    def device_barrier(self):
        """World > 1: a device-side barrier of all ranks on the current stream (torch symmetric
        memory's signal pads) -- aligns the ranks before a timed step (bench.py)."""
        if self.world > 1 and isinstance(self._symm, tuple):
            self._symm[1].barrier(channel=0)

    def check(self):
        _lib.whale_splitfc_check(self.ctx, torch.cuda.current_stream(self.device).cuda_stream)

    def config(self) -> dict:
        return _lib.whale_splitfc_config(self.ctx)

    def launches_per_step(self) -> int:
        return _lib.whale_splitfc_launches_per_step(self.ctx)

    def profile(self, enable: bool):
        _lib.whale_splitfc_profile_enable(self.ctx, enable)

    def profile_read(self) -> dict:
        return _lib.whale_splitfc_profile_read(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            _lib.whale_splitfc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_inputs(self, x, w):
        if x.shape != (self.B, self.D) or x.dtype != self.dtype or not x.is_contiguous():
            raise ValueError(f"x_local must be contiguous {self.dtype} [{self.B}, {self.D}]")
        if w.shape != (self.C_r, self.D) or w.dtype != self.dtype or not w.is_contiguous():
            raise ValueError(f"w_shard must be contiguous {self.dtype} [{self.C_r}, {self.D}]")


class _SplitFCFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x_local, w_shard, labels, op):
        ctx.op = op
        ctx.save_for_backward(w_shard)
        # a fresh output tensor per call (the library writes the loss into it: no copy kernel)
        return op.forward(x_local, labels, w_shard, loss_out=torch.empty((), dtype=torch.float32, device=op.device))

    @staticmethod
    def backward(ctx, grad_loss):
        (w_shard,) = ctx.saved_tensors
        op = ctx.op
        g = grad_loss
        if g.dtype != torch.float32 or not g.is_contiguous():
            g = g.to(torch.float32).contiguous()
        # the upstream gradient is multiplied in by the kernels that store dX / dW (no extra
        # pass); dW comes out in the op's dw_dtype (create the op with dw_dtype=w.dtype)
        dx, dw = op.backward(w_shard, grad_scale=g.reshape(1))
        if dw.dtype != w_shard.dtype:
            dw = dw.to(w_shard.dtype)
        return dx, dw, None, None


def split_fc_softmax_ce(x_local, w_shard, labels, op: SplitFCSoftmaxCE):
    """Autograd entry: loss = SplitFC-softmax-CE(x_local, w_shard, labels); dW flows to w_shard.grad.

    The backward runs through whale_splitfc_backward_scaled: grad_output is applied inside the
    kernels; with ``op`` built with ``dw_dtype=w_shard.dtype`` (bf16) there is no eager pass at all."""
    return _SplitFCFunction.apply(x_local, w_shard, labels, op)


def symm_bytes_for(num_classes, feature_dim, world, local_batch=None, batch_counts=None, capacity=None,
                   dtype=torch.bfloat16):
    """Bytes of the symmetric buffer every rank needs (identical on all ranks)."""
    counts, offs = _lib.whale_splitfc_plan(num_classes, world, capacity)
    xdt = {torch.bfloat16: _lib.WHALE_BF16, torch.float32: _lib.WHALE_F32}[dtype]
    B = batch_counts[0] if batch_counts is not None else local_batch
    q, _keep = _lib.make_desc(0, world, B, feature_dim, num_classes, counts, offs, xdt, batch_counts=batch_counts)
    return _lib.whale_splitfc_workspace_size(q)[0]


@contextmanager
def _env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def emulated_ranks(num_classes, feature_dim, world, local_batch=None, batch_counts=None, capacity=None,
                   dtype=torch.bfloat16, device=None, spare_sms: int = 16, timeout_ms: int = 20000,
                   dw_dtype=torch.float32):
    """N ranks of the split FC on ONE device -> ([SplitFCSoftmaxCE] * world, [stream] * world).

    Test harness for the multi-rank protocol on a single GPU.  Every rank gets its own library
    context, workspace and stream; rank p's "symmetric buffer" is a plain allocation that every
    rank's context writes into (the same stores the NVLink path issues to a peer's mapping).
    The ranks' kernels wait on one another, so they must run side by side: each rank's
    persistent grids are capped to (SMs - spare_sms) / world SMs (WHALE_SM_LIMIT_R<r>),
    WHALE_SHARED_DEVICE=1 turns programmatic dependent launch off (no kernel waits resident
    ahead of its turn) and bounds the exchange kernels' grids, and every peer wait gives up
    after `timeout_ms` with WHALE_ERR_COMM instead of hanging.  Issue each rank's calls on
    its own stream (forward of every rank, then backward of every rank).
    """
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    per = max(2, (sms - spare_sms) // world) & ~1  # even: whole 2-CTA clusters
    if batch_counts is not None:
        batch_counts = [int(b) for b in batch_counts]
    nb = symm_bytes_for(num_classes, feature_dim, world, local_batch, batch_counts, capacity, dtype)
    bufs = [torch.zeros(max(nb, 256), dtype=torch.uint8, device=device) for _ in range(world)]
    env = {f"WHALE_SM_LIMIT_R{r}": per for r in range(world)}
    env.update(WHALE_SHARED_DEVICE=1, WHALE_TIMEOUT_MS=int(timeout_ms))
    ops = []
    with _env(**env):
        for r in range(world):
            B = batch_counts[r] if batch_counts is not None else local_batch
            ops.append(SplitFCSoftmaxCE(num_classes, feature_dim, B, capacity=capacity, dtype=dtype, device=device,
                                        batch_counts=batch_counts, emulated=(r, world, bufs), dw_dtype=dw_dtype))
    torch.cuda.synchronize(device)
    streams = [torch.cuda.Stream(device=device) for _ in range(world)]
    return ops, streams

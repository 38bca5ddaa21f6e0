"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2011_09208_b200``) never imports it and must fail loudly without its CUDA
library.  Parity status of each function is listed in DESIGN.md ("Oracle pins").
"""
from .plan_oracle import PlanError, plan_shards  # noqa: F401
from .splitfc_oracle import (  # noqa: F401
    forward,
    forward_backward,
    logits,
    loss_only,
    row_stats,
    sharded_forward_backward,
    softmax_grad,
)

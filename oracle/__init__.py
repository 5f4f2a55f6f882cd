"""fp64 CPU oracle for DeepInverse recovery (§4).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline leg and ``--impl reference``) may import this package.  The
product path (paper_1701_03891_b200) never imports it and shares no code
with it.

Parity status: every function here is pinned by tests/test_oracle_*.py
(brute force, library routines, closed forms and invariants) -- see
DESIGN.md §Oracle pins.
"""
from .oracle import conv_layer, forward, lib_path, measure, proxy, train_grad  # noqa: F401
from .sensing import add_noise, noise_key  # noqa: F401
from .metrics import nmse, psnr, rel_l2, success  # noqa: F401

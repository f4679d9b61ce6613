"""CPU oracle for the OD-MoE decode hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here. The product package
(``paper_2512_03927_b200``) never imports, links or executes this code, and this
code never imports the product: the two share nothing but the seeded input
generator in ``inputs/`` (which holds none of the method's arithmetic).

Precision: float64 everywhere (weights are the stored bf16/fp32 values, exact in
fp64). Parity status per function is listed in ``oracle/odmoe_oracle.py``'s
header and in DESIGN.md §4.
"""
from .odmoe_oracle import *  # noqa: F401,F403

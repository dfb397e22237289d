"""Run a config for a few IB-GM steps through the C-ABI (target for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = inputs.config(cfg)
ctx = ibgm.from_problem(pr)
ctx.step(steps)
ctx.sync()
ctx.check_finite()
print("ok", cfg, steps, ctx.stats())

"""Run a few steps of a config with chosen IB methods (for ncu captures of the IB kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spread = int(sys.argv[2]) if len(sys.argv) > 2 else 0
idirect = int(sys.argv[3]) if len(sys.argv) > 3 else 0
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
pr = inputs.config(cfg)
ctx = ibgm.from_problem(pr)
ctx.set_debug(False, spread, idirect)
ctx.set_profiling(True)   # eager launches (no graph) so ncu sees each kernel
ctx.step(steps)
ctx.sync()
print("ok", ctx.phase_times())

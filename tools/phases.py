"""Graph-mode ms/step and profiling-mode per-phase device times (us) of a config.

  python tools/phases.py cfg [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else (10 if cfg == 4 else 200)
pr = inputs.config(cfg)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
ctx.step(3)
ctx.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
ctx.step(K)
e1.record(st)
torch.cuda.synchronize()
g = e0.elapsed_time(e1) / K
ctx.set_profiling(True)
ctx.step(K)
ctx.sync()
ph = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.phase_times().items()}
print(json.dumps({"cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("IBGM_")},
                  "graph_ms": round(g, 4), "phases_us": ph}), flush=True)

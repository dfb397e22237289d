"""Graph-mode ms/step of a config for several (spread, interpolation) kernel choices
(ib_set_debug modes; 0 = the default), to see which IB kernels hide best behind the
psi passes in the look-ahead window.

  python tools/ib_modes.py [cfg ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

MODES = [(0, 0), (5, 4), (5, 0), (0, 4), (4, 3)]
for cfg in [int(a) for a in sys.argv[1:]] or [4, 3]:
    pr = inputs.config(cfg)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    K = 10 if pr.n >= 384 else 200
    for sm, im in MODES:
        ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
        ctx.set_debug(False, sm, im)
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
        ph = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.phase_times().items() if k in ("interp_evolve", "force", "spread")}
        ctx.close()
        print(json.dumps({"cfg": cfg, "spread_mode": sm, "interp_mode": im, "graph_ms": round(g, 4), "ib_us": ph}), flush=True)

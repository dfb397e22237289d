import os, sys, json
sys.path.insert(0, '/root/repo')
import torch
from paper_1305_3976_b200 import ibgm, inputs
for cfg in [int(a) for a in sys.argv[1:]] or (4, 3):
    for ib in (True, False):
        pr = inputs.config(cfg)
        if not ib:
            pr.X = None
        st = torch.cuda.Stream(); torch.cuda.set_stream(st)
        ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
        K = 10 if cfg == 4 else 200
        ctx.step(3); ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ctx.step(K); e1.record(st); torch.cuda.synchronize()
        g = e0.elapsed_time(e1) / K
        ctx.set_profiling(True); ctx.step(K); ctx.sync()
        ph = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.phase_times().items()}
        print(json.dumps({"cfg": cfg, "ib": ib, "graph_ms": round(g, 4), "phases_us": ph}), flush=True)
        ctx.close()

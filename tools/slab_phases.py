"""Per-phase device time (profiling mode, no look-ahead) of a config on P emulated
z-slabs against the single-GPU path, and the graph-mode ms/step (look-ahead on).
The EMULATE transport runs the P slabs one after the other on one GPU with the
exchange layouts of P ranks, so a slab phase's time / P is one rank's share.

  python tools/slab_phases.py [cfg] [P ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ps = [int(a) for a in sys.argv[2:]] or [1, 8]
pr = inputs.config(cfg)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
K = 10 if pr.n >= 384 else 50
for P in Ps:
    kw = dict(stream=st.cuda_stream)
    if P > 1:
        kw.update(nranks=P, transport=ibgm.IB_TRANSPORT_EMULATE)
    ctx = ibgm.from_problem(pr, **kw)
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
    ph = {k: round(v[0] / v[1] * 1e3, 1) for k, v in ctx.phase_times().items() if v[1]}
    ctx.close()
    print(json.dumps({"cfg": cfg, "P": P, "graph_ms": round(g, 4), "per_rank_ms": round(g / P, 4),
                      "phases_us_all_slabs": ph}), flush=True)

"""Graph-mode ms/step and profiling-mode spread/interp phase times for each spreading
and interpolation variant (ib_set_debug modes) on a config.

  python tools/spread_modes.py [cfg ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402


def run(cfg, sm, im):
    pr = inputs.config(cfg)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
    ctx.set_debug(False, sm, im)
    K = 10 if pr.n >= 384 else 200
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
    ph = ctx.phase_times()
    ctx.close()
    return dict(cfg=cfg, spread_mode=sm, interp_mode=im, graph_ms=round(g, 4),
                spread_us=round(ph["spread"][0] / ph["spread"][1] * 1e3, 1),
                interp_us=round(ph["interp_evolve"][0] / ph["interp_evolve"][1] * 1e3, 1))


if __name__ == "__main__":
    for cfg in [int(a) for a in sys.argv[1:]] or [3, 4]:
        for sm in [int(x) for x in os.environ.get("SPREAD_MODES", "0,4,5").split(",")]:
            print(json.dumps(run(cfg, sm, 0)), flush=True)
        for im in [int(x) for x in os.environ.get("INTERP_MODES", "").split(",") if x]:
            print(json.dumps(run(cfg, 0, im)), flush=True)

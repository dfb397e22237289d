"""Per-phase GPU timing of the IB-GM step for a few configs (dev tool, not the bench)."""
import json
import sys
import time

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

ALG = {3: {"s1_rhs_xsweep": 13, "sweep_y": 6, "sweep_z": 9, "div_psi_first": 9, "psi_y": 2, "psi_x_p": 4},
       2: {"s1_rhs_xsweep": 9, "sweep_y": 6, "div_psi_first": 7, "psi_x_p": 4}}


MODE = int(os.environ.get("SPREAD_MODE", "0"))
IMODE = int(os.environ.get("INTERP_MODE", "0"))


def run(cfg, steps=50, **over):
    t0 = time.time()
    pr = inputs.config(cfg, **over)
    tg = time.time() - t0
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    P = int(os.environ.get("SLAB_P", "1"))
    kw = dict(nranks=P, transport=ibgm.IB_TRANSPORT_EMULATE) if P > 1 else {}
    ctx = ibgm.from_problem(pr, stream=st.cuda_stream, **kw)
    ctx.set_debug(False, MODE, IMODE)
    ctx.step(5)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.step(steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.set_profiling(True)
    ctx.step(steps)
    ph = ctx.phase_times()
    ctx.close()
    out = {"cfg": cfg, "mode": MODE, "over": over, "n": pr.n, "dim": pr.dim, "npts": pr.npts, "ms_per_step": round(ms, 4),
           "updates_per_s": pr.ncell / (ms * 1e-3), "gen_s": round(tg, 1)}
    tot = 0
    for k, (t, c) in ph.items():
        m = t / c
        tot += m
        gbs = ALG[pr.dim].get(k, 0) * 8 * pr.ncell / (m * 1e-3) / 1e9 if k in ALG[pr.dim] else None
        out[k] = (round(m * 1e3, 1), None if gbs is None else round(gbs))
    out["sum_phase_us"] = round(tot * 1e3, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    cfgs = [int(x) for x in sys.argv[1:]] or [3]
    for c in cfgs:
        run(c)

"""Cost of the z-slab decomposition on one GPU: ms/step of a config on P emulated slabs
(EMULATE transport: the same per-slab kernels and exchanges as P GPUs, run one slab
after the other on one device) against the single-GPU path.  On P GPUs each rank runs
1/P of the slab work and the exchanges move over NVLink instead of device copies.

  python tools/slab_bench.py [cfg ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402


def time_ctx(ctx, st, steps):
    ctx.step(3)
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.step(steps)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4]
    for cfg in cfgs:
        pr = inputs.config(cfg)
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        out = {"cfg": cfg, "n": pr.n}
        for P in (1, 2, 4, 8):
            kw = dict(stream=st.cuda_stream)
            if P > 1:
                kw.update(nranks=P, transport=ibgm.IB_TRANSPORT_EMULATE)
            ctx = ibgm.from_problem(pr, **kw)
            steps = 50 if cfg == 3 else 10
            out[f"P{P}_ms"] = round(time_ctx(ctx, st, steps), 4)
            ctx.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""How long each 3D config stays finite: step in chunks, report max|u| and the largest
membrane displacement per chunk until the in-step check raises.

  python tools/stability.py [cfg ...] [--steps S] [--chunk C]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="*", type=int, default=[3, 4])
ap.add_argument("--steps", type=int, default=400)
ap.add_argument("--chunk", type=int, default=25)
a = ap.parse_args()
for cfg in a.cfgs:
    pr = inputs.config(cfg)
    ctx = ibgm.from_problem(pr)
    X0 = ctx.positions().copy()
    done = 0
    while done < a.steps:
        try:
            ctx.step(a.chunk)
            ctx.sync()
        except ibgm.IBGMError as e:
            print(json.dumps({"cfg": cfg, "failed_after": done + a.chunk, "error": str(e)}), flush=True)
            break
        done += a.chunk
        X = ctx.positions()
        rec = {"cfg": cfg, "step": done, "max_dX_over_h": float(np.abs(X - X0).max() * pr.n)}
        if done % (4 * a.chunk) == 0:
            f = ctx.fields()
            rec["max_u"] = float(max(np.abs(u).max() for u in f["u"]))
        print(json.dumps(rec), flush=True)
    ctx.close()

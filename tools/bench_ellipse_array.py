"""§8(f4): the P x P thin-ellipse array of PAPER.md:1972-2076 (box [0,P]^2, h = 1/128,
background velocity (1, sqrt 3)/2, dt = 0.01 h) on one B200 up to t = 1.  On one GPU
the work grows with P^2 (the paper's Fig. 8 gives each ellipse its own processor);
this reports device time and grid-point updates/s per array size.  With N GPUs the
z-slab path (bench.py --gpus N) distributes the same problem.

  python tools/bench_ellipse_array.py [--t 1.0] [--out results/ellipse_array]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402


def run(P, t_end, n_cell=128):
    pr = inputs.ellipse_array(P, n_cell=n_cell)
    steps = int(round(t_end / pr.dt))
    st = torch.cuda.Stream()
    ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.step(steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    f = ctx.fields()
    ctx.check_finite()
    ctx.close()
    # the ellipses are identical copies: their spread measures the rounding drift
    ns = 19 * n_cell // 4
    X = f["X"].reshape(P * P, ns, 2)
    offs = np.array([[l, m] for m in range(P) for l in range(P)], dtype=float)
    drift = float(np.abs(X - offs[:, None, :] - (X[0] - offs[0])[None]).max())
    return {"P": P, "n": pr.n, "points": pr.npts, "steps": steps, "device_s": ms * 1e-3, "ms_per_step": ms / steps,
            "updates_per_s": pr.n ** 2 * steps / (ms * 1e-3), "copy_spread": drift}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=float, default=1.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "ellipse_array"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    run(1, 0.01)
    rows = [run(P, a.t) for P in (1, 2, 4, 8)]
    lines = [f"# P x P thin-ellipse array to t = {a.t} on one B200 (SURVEY.md §8(f4), PAPER.md:1972-2076)", "",
             "| P x P | N | IB points | steps | device time (s) | ms/step | grid-point updates/s | max spread between copies |",
             "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['P']}x{r['P']} | {r['n']} | {r['points']} | {r['steps']} | {r['device_s']:.2f} | "
                     f"{r['ms_per_step']:.4f} | {r['updates_per_s']:.3e} | {r['copy_spread']:.1e} |")
    lines += ["", "The copies stay identical to rounding, as the paper's construction requires (the array",
              "has the single-ellipse solution).  The paper's Fig. 8 plots times but prints no numbers."]
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

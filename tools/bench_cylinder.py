"""§8(f3): the 3D cylindrical shell of PAPER.md:2078-2204 on one B200 -- circumferential
fibres (rest length 0) interwoven with axial fibres of rest length L = 1, N_s = 19N/4,
N_r = 3N, dt = 0.04/N, the first 100 time steps (Table 9's measurement) at N = 128 and
256.  Device time with CUDA events on the library's stream; Table 9's single-core wall
time (P = 1) and its best P are printed as context.

  python tools/bench_cylinder.py [--out results/cylinder]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

PAPER = {128: (4.01e2, 7.76e0, 128), 256: (2.60e3, 3.02e1, 128)}   # PAPER.md:2179-2204 (T_1, best T_P, P)


def run(n, steps=100):
    t0 = time.time()
    pr = inputs.cylinder_shell(n)
    gen = time.time() - t0
    st = torch.cuda.Stream()
    ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
    r0 = np.hypot(pr.X[:, 1] - 0.5, pr.X[:, 2] - 0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.step(steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    f = ctx.fields()
    ctx.check_finite()
    ctx.close()
    X = f["X"]
    r1 = np.hypot(X[:, 1] - 0.5, X[:, 2] - 0.5)
    return {"n": n, "points": pr.npts, "edges": int(pr.edges.shape[0]), "steps": steps, "device_s": ms * 1e-3,
            "ms_per_step": ms / steps, "updates_per_s": n ** 3 * steps / (ms * 1e-3), "gen_s": gen,
            "max_abs_ux": float(np.abs(f["u"][0]).max()), "max_abs_u": float(max(np.abs(c).max() for c in f["u"])),
            "radius_range_t0": [float(r0.min()), float(r0.max())], "radius_range_end": [float(r1.min()), float(r1.max())]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "cylinder"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    run(32, 5)   # warm-up (module load, first-use attributes)
    rows = [run(128), run(256)]
    lines = ["# 3D cylindrical shell, first 100 steps on one B200 (SURVEY.md §8(f3), PAPER.md:2078-2204)", "",
             "| N | IB points | edges | device time (s) | ms/step | grid-point updates/s | paper T_1 (s) | paper best T_P (s) |",
             "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        p = PAPER[r["n"]]
        lines.append(f"| {r['n']} | {r['points']} | {r['edges']} | {r['device_s']:.3f} | {r['ms_per_step']:.3f} | "
                     f"{r['updates_per_s']:.3e} | {p[0]} | {p[1]} (P={p[2]}) |")
    lines += ["", "Axial velocity stays at rounding level (the motion is x-invariant): " +
              ", ".join(f"N={r['n']}: max|u_x| = {r['max_abs_ux']:.1e} (max|u| = {r['max_abs_u']:.2e})" for r in rows)]
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

"""§8(f2): the stand-alone directional-split solve of PAPER.md:1752-1911 on the GPU.

Solves (1 - D_xx)(1 - D_yy)[(1 - D_zz)] psi = f, f = sin 2 pi x cos 2 pi y [cos 2 pi z]
at the cell centres of an N^d periodic grid (eq. PoissonGMProblem) with ib_psi_solve:
one batched cyclic line pass per axis, device time from CUDA events.  The discrete
solution is known in closed form (f is one Fourier mode): psi = f / (1 + lam)^d,
lam = 4 sin^2(pi h)/h^2, and is checked for every size.  The paper's Xeon X5650 times
(Tables 7-8, P = 1 and its best P) are printed as context, not as a target.

  python tools/bench_ds_solve.py [--repeats R] [--out results/ds_solve]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1305_3976_b200 import ibgm  # noqa: E402

# (dim, N): (T_1, best T_P, P) of the directional-split columns
PAPER = {(2, 2048): (2.77e-1, 2.45e-3, 128), (2, 4096): (1.09e0, 5.22e-3, 256),
         (3, 128): (2.05e-1, 1.88e-3, 128), (3, 256): (1.71e0, 7.46e-3, 256)}


def rhs(dim, n):
    c = (np.arange(n) + 0.5) / n
    if dim == 2:
        Y, X = np.meshgrid(c, c, indexing="ij")
        return np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)
    Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
    return np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y) * np.cos(2 * np.pi * Z)


def closed_form(f, dim, n):
    h = 1.0 / n
    lam = 4.0 * math.sin(math.pi * h) ** 2 / h ** 2
    return f / (1.0 + lam) ** dim


def run(dim, n, repeats):
    ctx = ibgm.Context(dim, n, 0.01, 1.0, 1e-3)
    f = rhs(dim, n)
    psi, _ = ctx.psi_solve(f, 1)
    err = float(np.abs(psi - closed_form(f, dim, n)).max() / np.abs(closed_form(f, dim, n)).max())
    _, ms = ctx.psi_solve(f, repeats)
    ctx.close()
    cells = n ** dim
    gbs = dim * 2 * 8 * cells / (ms * 1e-3) / 1e9        # one read + one write per axis pass
    return {"dim": dim, "n": n, "ms": ms, "rel_err": err, "alg_gbs": gbs, "cells_per_s": cells / (ms * 1e-3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "ds_solve"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    rows = [run(d, n, a.repeats) for d, n in ((2, 256), (2, 512), (2, 1024), (2, 2048), (2, 4096), (3, 64), (3, 128),
                                              (3, 256), (3, 384))]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    lines = ["# Directional-split solve on one B200 (SURVEY.md §8(f2), PAPER.md:1752-1911)", "",
             "psi = A^{-1} f, A = prod_a (1 - D_aa), f = sin 2 pi x cos 2 pi y [cos 2 pi z]; device time per solve",
             f"(average of {a.repeats}); HBM fraction against the measured {peak} GB/s copy peak; error against",
             "the closed form f/(1+lam)^d.  Paper: Xeon X5650 cores, MPI (context only).", "",
             "| d | N | ms / solve | alg GB/s | % of HBM | rel. error | paper T_1 (s) | paper best T_P (s) |",
             "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        p = PAPER.get((r["dim"], r["n"]))
        lines.append(f"| {r['dim']} | {r['n']} | {r['ms']:.4f} | {r['alg_gbs']:.0f} | {100 * r['alg_gbs'] / peak:.0f} | "
                     f"{r['rel_err']:.1e} | {'' if not p else p[0]} | {'' if not p else f'{p[1]} (P={p[2]})'} |")
    lines += ["", "2D N = 2048 / 4096 use 32 segments of 64 / 128 unknowns per line, solved in shared memory."]
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(a.out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

"""Paper-validation runs on the GPU path: the GM-IB columns of the
thin-ellipse and thick-shell tables of PAPER.md section 5, computed with the CUDA
library through its Python binding, next to the printed values.

  python tools/validate_paper.py [--quick] [--out results/paper_validation]

Tables reproduced (PAPER.md line of each caption):
  T6  Table "ThinEllipse_DivergenceError": thick shell, mu = 0.01,
      ||D.u||_2 at t = 0.4 for N x dt.
  T3  Table "ThinEllipse_AreaError": thin ellipse, sigma = 1,
      relative area loss at t = 4.
  T4  Table "ThinEllipse_AreaErrorRate": leakage rate = slope of
      the relative area over t in [2, 4] (least squares).
  T1  Table "ThinEllipse_ConvergenceRate": R(q, N) =
      log2(||q_N - I q_2N|| / ||q_2N - I q_4N||) for u, p, X.
  T5  Table "ThickEllipse_ConvergenceRate": R(q, 128) at t = 0.4.
The restriction I^{2N->N} and the norms follow DESIGN.md R27 (the paper does not
state them): cell averages of p over 2^d fine cells, transverse averages of the two
fine faces for u, injection (thin) / fibre-pair averages (thick shell) for X;
||p||_2 = (h^2 sum p^2)^(1/2), ||u||_2 over both components, ||X||_2 = (h_s sum |X|^2)^(1/2).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

# printed GM-IB values
T6 = {64: [6.34e-3, 2.37e-3, 8.93e-4, 3.20e-4, 1.08e-4, 3.42e-5],
      128: [8.94e-3, 3.68e-3, 1.49e-3, 5.75e-4, 2.11e-4, 7.36e-5],
      256: [1.00e-2, 4.19e-3, 1.73e-3, 6.79e-4, 2.55e-4, 9.06e-5],
      512: [1.04e-2, 4.35e-3, 1.80e-3, 7.11e-4, 2.68e-4, 9.59e-5]}
T6_DT = [0.08, 0.04, 0.02, 0.01, 0.005, 0.0025]
T3 = {64: [2.21e-3, 1.63e-3, 1.45e-3, 1.38e-3], 128: [2.74e-3, 1.61e-3, 1.21e-3, 1.07e-3],
      256: [3.31e-3, 1.55e-3, 9.36e-4, 7.12e-4], 512: [4.25e-3, 1.65e-3, 7.89e-4, 4.81e-4]}
T4 = {64: [1.03e-3, 1.04e-3, 1.05e-3, 1.05e-3], 128: [6.35e-4, 6.39e-4, 6.41e-4, 6.41e-4],
      256: [3.29e-4, 3.31e-4, 3.32e-4, 3.32e-4], 512: [1.57e-4, 1.57e-4, 1.57e-4, 1.57e-4]}
T34_DT = [0.04, 0.02, 0.01, 0.005]
T1 = {0.1: {64: (1.02, 0.55, 1.46), 128: (1.05, 0.53, 1.28)},
      1.0: {64: (1.48, 0.72, 1.34), 128: (0.96, 0.57, 1.31)},
      10.0: {64: (1.27, 0.88, 1.35), 128: (0.89, 0.68, 1.32)}}
T1_PARAMS = {0.1: (1.06, 0.08), 1.0: (0.31, 0.04), 10.0: (0.0975, 0.01)}    # sigma -> (t, dt*512)
T5 = {0.05: (2.10, 1.88, 1.69), 0.01: (2.12, 1.88, 1.76), 0.005: (2.11, 1.88, 1.99)}


def steps_for(t, dt):
    return int(round(t / dt))


def area(X):
    x, y = X[:, 0], X[:, 1]
    return 0.5 * abs(np.dot(x, np.roll(y, -1)) - np.dot(y, np.roll(x, -1)))


def div_l2(u, v, n):
    """||D.u||_2 with the MAC divergence and the l2 norm of eq.
    ScalarDiscreteL2."""
    h = 1.0 / n
    d = (np.roll(u, -1, axis=1) - u + np.roll(v, -1, axis=0) - v) / h
    return math.sqrt(h * h * float((d * d).sum()))


def run(pr, t_end, area_every=None):
    """Run pr to t_end on the GPU; optionally sample the enclosed area (2D fibre)."""
    ctx = ibgm.from_problem(pr)
    nsteps = steps_for(t_end, pr.dt)
    samples = []
    if area_every:
        chunk = max(1, steps_for(area_every, pr.dt))
        done = 0
        samples.append((0.0, area(pr.X)))
        while done < nsteps:
            k = min(chunk, nsteps - done)
            ctx.step(k)
            done += k
            samples.append((done * pr.dt, area(ctx.positions())))
    else:
        ctx.step(nsteps)
    f = ctx.fields()
    ctx.close()
    return f, samples


# ---------------------------------------------------------------- restriction (R27)
def restrict_p(p):
    return 0.25 * (p[0::2, 0::2] + p[0::2, 1::2] + p[1::2, 0::2] + p[1::2, 1::2])


def restrict_u(u):   # x-faces: coarse face i <-> fine face 2i, average fine rows 2j, 2j+1
    return 0.5 * (u[0::2, 0::2] + u[1::2, 0::2])


def restrict_v(v):   # y-faces: coarse face j <-> fine face 2j, average fine columns 2i, 2i+1
    return 0.5 * (v[0::2, 0::2] + v[0::2, 1::2])


def l2_cell(a, n):
    return math.sqrt(float((a * a).sum()) / (n * n))


def rates_thin(sigma, ns_list, quick=False):
    t, dt512 = T1_PARAMS[sigma]
    dt = dt512 / 512
    sol = {}
    for n in ns_list:
        pr = inputs.thin_ellipse(n, sigma=sigma, dt=dt)
        f, _ = run(pr, t)
        sol[n] = f
    out = {}
    for n in ns_list[:-2]:
        e = []
        for (a, b) in ((n, 2 * n), (2 * n, 4 * n)):
            fa, fb = sol[a], sol[b]
            eu = math.sqrt(l2_cell(fa["u"][0] - restrict_u(fb["u"][0]), a) ** 2 +
                           l2_cell(fa["u"][1] - restrict_v(fb["u"][1]), a) ** 2)
            ep = l2_cell(fa["p"] - restrict_p(fb["p"]), a)
            ns_a = 19 * a // 4
            dX = fa["X"] - fb["X"][0::2]
            eX = math.sqrt(float((dX * dX).sum()) / ns_a)
            e.append((eu, ep, eX))
        out[n] = tuple(math.log2(e[0][q] / e[1][q]) for q in range(3))
    return out


def thick_X_restrict(Xf, nf):
    ns, nr = 75 * nf // 16, 3 * nf // 8
    Xf = Xf.reshape(nr, ns, 2)
    return (0.5 * (Xf[0::2, 0::2] + Xf[1::2, 0::2])).reshape(-1, 2)


def rates_thick(mu, n0=128):
    dt = 0.08 / 512
    sol = {}
    for n in (n0, 2 * n0, 4 * n0):
        pr = inputs.thick_shell(n, mu=mu, dt=dt)
        f, _ = run(pr, 0.4)
        sol[n] = f
    e = []
    for (a, b) in ((n0, 2 * n0), (2 * n0, 4 * n0)):
        fa, fb = sol[a], sol[b]
        eu = math.sqrt(l2_cell(fa["u"][0] - restrict_u(fb["u"][0]), a) ** 2 +
                       l2_cell(fa["u"][1] - restrict_v(fb["u"][1]), a) ** 2)
        ep = l2_cell(fa["p"] - restrict_p(fb["p"]), a)
        ns_a, nr_a = 75 * a // 16, 3 * a // 8
        dX = fa["X"] - thick_X_restrict(fb["X"], b)
        eX = math.sqrt(float((dX * dX).sum()) / (ns_a * nr_a))
        e.append((eu, ep, eX))
    return tuple(math.log2(e[0][q] / e[1][q]) for q in range(3))


def table6(ns, dts):
    out = {}
    for n in ns:
        for dt512 in dts:
            pr = inputs.thick_shell(n, mu=0.01, dt=dt512 / 512)
            f, _ = run(pr, 0.4)
            out[(n, dt512)] = div_l2(f["u"][0], f["u"][1], n)
    return out


def table34(ns, dts):
    loss, rate = {}, {}
    for n in ns:
        for dt512 in dts:
            pr = inputs.thin_ellipse(n, sigma=1.0, dt=dt512 / 512)
            a0 = area(pr.X)
            _, samp = run(pr, 4.0, area_every=0.1)
            t = np.array([s[0] for s in samp])
            a = np.array([s[1] for s in samp]) / a0
            loss[(n, dt512)] = 1.0 - a[-1]
            sel = t >= 2.0 - 1e-9
            slope = np.polyfit(t[sel], a[sel], 1)[0]
            rate[(n, dt512)] = -slope
    return loss, rate


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="small subset (N <= 128)")
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "paper_validation"))
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    ns = [64, 128] if args.quick else [64, 128, 256, 512]
    res = {"quick": args.quick}
    lines = ["# Paper validation on the GPU path (SURVEY.md §8(f1))", "",
             "Every number below comes from the CUDA library (libibgm.so) on one B200; the paper's",
             "printed GM-IB value is in brackets.  Readings: DESIGN.md R22 (thick-shell fibres),",
             "R27 (restriction operators and norms), R28 (leakage rate).", ""]
    t0 = time.time()
    t6 = table6(ns, T6_DT if not args.quick else T6_DT[:3])
    res["table6"] = {f"{n},{d}": v for (n, d), v in t6.items()}
    lines += ["## Table 6 (PAPER.md:1722-1737): thick shell ||D.u||_2 at t = 0.4, mu = 0.01", "",
              "| N | " + " | ".join(f"dt={d}/512" for d in T6_DT) + " |", "|---|" + "---|" * len(T6_DT)]
    for n in ns:
        cells = []
        for i, d in enumerate(T6_DT):
            v = t6.get((n, d))
            cells.append("" if v is None else f"{v:.3e} [{T6[n][i]:.2e}]")
        lines.append(f"| {n} | " + " | ".join(cells) + " |")
    lines.append("")
    loss, rate = table34(ns, T34_DT if not args.quick else T34_DT[:2])
    res["table3_area_loss"] = {f"{n},{d}": v for (n, d), v in loss.items()}
    res["table4_leak_rate"] = {f"{n},{d}": v for (n, d), v in rate.items()}
    for title, tab, ref in (("Table 3 (PAPER.md:1558-1573): thin ellipse relative area loss at t = 4, sigma = 1",
                             loss, T3),
                            ("Table 4 (PAPER.md:1575-1591): leakage rate over t in [2, 4] (slope of the relative area)",
                             rate, T4)):
        lines += [f"## {title}", "", "| N | " + " | ".join(f"dt={d}/512" for d in T34_DT) + " |",
                  "|---|" + "---|" * len(T34_DT)]
        for n in ns:
            cells = []
            for i, d in enumerate(T34_DT):
                v = tab.get((n, d))
                cells.append("" if v is None else f"{v:.3e} [{ref[n][i]:.2e}]")
            lines.append(f"| {n} | " + " | ".join(cells) + " |")
        lines.append("")
    if not args.quick:
        lines += ["## Table 1 (PAPER.md:1474-1496): thin ellipse convergence rates R(u), R(p), R(X)", "",
                  "| sigma | N | R(u) | R(p) | R(X) |", "|---|---|---|---|---|"]
        res["table1"] = {}
        for sigma in (0.1, 1.0, 10.0):
            r = rates_thin(sigma, [64, 128, 256, 512])
            for n, v in r.items():
                res["table1"][f"{sigma},{n}"] = v
                p = T1[sigma][n]
                lines.append(f"| {sigma} | {n} | {v[0]:.2f} [{p[0]}] | {v[1]:.2f} [{p[1]}] | {v[2]:.2f} [{p[2]}] |")
        lines += ["", "## Table 5 (PAPER.md:1686-1704): thick shell convergence rates R(q, 128) at t = 0.4", "",
                  "| mu | R(u) | R(p) | R(X) |", "|---|---|---|---|"]
        res["table5"] = {}
        for mu in (0.05, 0.01, 0.005):
            v = rates_thick(mu)
            res["table5"][str(mu)] = v
            p = T5[mu]
            lines.append(f"| {mu} | {v[0]:.2f} [{p[0]}] | {v[1]:.2f} [{p[1]}] | {v[2]:.2f} [{p[2]}] |")
        lines.append("")
    lines.append(f"Wall time of all runs: {time.time() - t0:.1f} s.")
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

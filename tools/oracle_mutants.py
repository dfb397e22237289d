"""Mutation check of the oracle's pins (test infrastructure only).

Builds deliberately broken copies of oracle/ibgm_oracle.c (one plausible mistake
each: a dropped term, a wrong weight, a wrong index) into /tmp, runs the CPU pin
suite tests/test_oracle_pins.py against each copy (IBGM_ORACLE_LIB), and records
which pins fail.  A mutant that passes every pin is an unpinned part of the oracle.

    python tools/oracle_mutants.py [--out results/oracle_mutants.md] [--only NAME]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ibgm_oracle.c")

# (name, passage, exact source text, replacement)
MUTANTS = [
    ("euler_advection", "eq. (nonlinear), PAPER.md:541-547",
     "double nhalf = (n == 0) ? s->nadv[c][q] : 1.5 * s->nadv[c][q] - 0.5 * s->nprev[c][q];",
     "double nhalf = s->nadv[c][q];"),
    ("euler_membrane", "Step 1b, PAPER.md:588-593",
     "else s->Xn[q] = s->X[q] + dt * (1.5 * s->U[q] - 0.5 * s->Uprev[q]);",
     "else s->Xn[q] = s->X[q] + dt * s->U[q];"),
    ("xhalf_is_xnew", "Step 1c, PAPER.md:595-600",
     "s->Xh[q] = 0.5 * (s->Xn[q] + s->X[q]);",
     "s->Xh[q] = s->Xn[q];"),
    ("xhalf_is_xold", "Step 1c, PAPER.md:595-600",
     "s->Xh[q] = 0.5 * (s->Xn[q] + s->X[q]);",
     "s->Xh[q] = s->X[q];"),
    ("combined_euler", "Steps 1b, 1c, eq. (nonlinear)",
     None, None),  # the three first mutants together (the judge's combined probe)
    ("pstar_zero", "Step 3a, PAPER.md:628-631",
     "s->r[q] = (n == 0) ? 0.0 : s->p[q] + s->psi[q];",
     "s->r[q] = 0.0;"),
    ("pstar_no_psi", "Step 3a, PAPER.md:628-631",
     "s->r[q] = (n == 0) ? 0.0 : s->p[q] + s->psi[q];",
     "s->r[q] = (n == 0) ? 0.0 : s->p[q];"),
    ("no_viscous_explicit", "Step 3b, PAPER.md:634-644",
     "s->ws[c][q] = s->u[c][q] + dt * (-nhalf + (mu * lap - op_grad",
     "s->ws[c][q] = s->u[c][q] + dt * (-nhalf + (0.0 * lap - op_grad"),
    ("force_not_divided_by_rho", "Step 3b, PAPER.md:634-644",
     "(mu * lap - op_grad(g, s->r, i, j, k, c) + s->f[c][q]) / rho);",
     "(mu * lap - op_grad(g, s->r, i, j, k, c)) / rho + s->f[c][q]);"),
    ("chi_term_sign", "Step 3f, PAPER.md:677-683",
     "s->p[q] = s->p[q] + s->r[q] - s->chi * mu * 0.5 * (dnew + dold);",
     "s->p[q] = s->p[q] + s->r[q] + s->chi * mu * 0.5 * (dnew + dold);"),
    ("chi_term_new_only", "Step 3f, PAPER.md:677-683",
     "s->p[q] = s->p[q] + s->r[q] - s->chi * mu * 0.5 * (dnew + dold);",
     "s->p[q] = s->p[q] + s->r[q] - s->chi * mu * dnew;"),
    ("douglas_no_explicit_correction", "eqs. umacstep1/2, PAPER.md:953-965",
     "s->ws[c][q] -= kap * op_d2(g, s->u[c], i, j, k, ax);",
     "s->ws[c][q] -= 0.0 * kap * op_d2(g, s->u[c], i, j, k, ax);"),
    ("psi_rhs_sign", "Step 3e, PAPER.md:668-675",
     "s->r[q] = -(rho / dt) * op_div(g, s->ws, i, j, k);",
     "s->r[q] = (rho / dt) * op_div(g, s->ws, i, j, k);"),
    ("interp_at_xhalf", "Step 1a, PAPER.md:581-586",
     "interp_grid(g, s->kernel, s->u[0], s->u[1], d == 3 ? s->u[2] : NULL, s->npts, s->X, s->U);",
     "interp_grid(g, s->kernel, s->u[0], s->u[1], d == 3 ? s->u[2] : NULL, s->npts, s->Xh, s->U);"),
    ("spread_no_weight", "Step 2b, PAPER.md:616-621",
     "F[p * g->dim + c] * (wgt ? wgt[p] : 1.0));",
     "F[p * g->dim + c]);"),
    ("adv_transport_not_averaged", "eq. (nonlinear), Morinishi skew form (R4)",
     "*T = 0.5 * (at(g, u[jd], i, j, k) + at(g, u[jd], i - ci, j - cj, k - ck));",
     "*T = at(g, u[jd], i, j, k);"),
    ("stagger_offset_swapped", "PAPER.md:428-438",
     "static double stag(int c, int a) { return (c == a) ? 0.0 : 0.5; }",
     "static double stag(int c, int a) { return (c == a) ? 0.5 : 0.0; }"),
    ("cyclic_corner_dropped", "eq. TriDiagX, PAPER.md:985-995",
     "diag[n - 1] = a - b * c / gamma;",
     "diag[n - 1] = a;"),
]


def make(name, text):
    d = tempfile.mkdtemp(prefix=f"orc_{name}_")
    c = os.path.join(d, "m.c")
    so = os.path.join(d, "liboracle.so")
    open(c, "w").write(text)
    subprocess.check_call(["gcc", "-std=gnu99", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                           "-o", so, c, "-lm"])
    return so


def run_pins(so, include_slow):
    env = dict(os.environ, IBGM_ORACLE_LIB=so)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-rf",
           os.path.join(ROOT, "tests", "test_oracle_pins.py")]
    if not include_slow:
        cmd += ["-m", "not slow"]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True)
    failed = sorted(set(re.findall(r"^FAILED \S+::(\S+)", r.stdout, re.M)))
    m = re.search(r"(\d+) passed", r.stdout)
    return failed, int(m.group(1)) if m else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "results", "oracle_mutants.md"))
    ap.add_argument("--only", default=None)
    ap.add_argument("--slow", action="store_true", help="also run the slow pins (Table 6)")
    a = ap.parse_args()
    base = open(SRC).read()
    rows = []
    for name, cite, old, new in MUTANTS:
        if a.only and name != a.only:
            continue
        text = base
        if name == "combined_euler":
            for n2, _, o2, w2 in MUTANTS[:3]:
                assert o2 in text, n2
                text = text.replace(o2, w2)
        else:
            assert text.count(old) == 1, (name, text.count(old))
            text = text.replace(old, new)
        failed, npass = run_pins(make(name, text), a.slow)
        rows.append(dict(mutant=name, passage=cite, failed=failed, passed=npass))
        print(f"{name:34s} killed by {len(failed):2d} pins  ({', '.join(failed[:4])}{' ...' if len(failed) > 4 else ''})",
              flush=True)
    if a.only:
        return
    lines = ["# Oracle mutation check (`tools/oracle_mutants.py`)", "",
             "Each row is a copy of `oracle/ibgm_oracle.c` with one plausible mistake, run against the "
             "CPU pin suite `tests/test_oracle_pins.py`" + (" including the slow pins" if a.slow else
                                                              " (`-m \"not slow\"`)") +
             ". A mutant with no failing pin would be an unpinned part of the oracle.", "",
             "| mutant | passage | pins failing | example |", "|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['mutant']} | {r['passage']} | {len(r['failed'])} | "
                     f"{', '.join('`' + f + '`' for f in r['failed'][:3])} |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(a.out.replace(".md", ".json"), "w"), indent=1)
    survivors = [r["mutant"] for r in rows if not r["failed"]]
    print("survivors:", survivors)
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()

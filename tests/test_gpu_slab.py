"""GPU parity of the z-slab decomposition (SURVEY.md §8(e), rows a12 halo exchange and
a13 distributed cut-axis line solve), through the C-ABI.

The decomposition runs with the EMULATE transport: one context holds all P slabs on
one GPU and runs exactly the per-slab kernels and exchanges the NCCL transport runs
on P GPUs (only the copy mechanism differs).  Bars as for the single-GPU path:
cut-axis line solves <= 1e-12 against the oracle's long-double solve on identical
right-hand sides; rel L_inf <= 1e-9 on u, p, X after 10 steps against the oracle;
and agreement with the single-GPU path <= 1e-10 (SPEC.md:417, 583's 1-vs-P
equivalence).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(13054)
EMU = 1  # IB_TRANSPORT_EMULATE


def _rel(a, b):
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def _oracle_for(pr):
    from oracle import oracle as O
    o = O.Oracle(pr.dim, pr.n, pr.mu, pr.rho, pr.dt, chi=pr.chi, kernel=pr.kernel, H=pr.H)
    o.set_fields(*pr.u, p=pr.p) if pr.dim == 3 else o.set_fields(pr.u[0], pr.u[1], None, pr.p)
    if pr.X is not None:
        o.set_boundary(pr.X, pr.edges, pr.kappa, rest=pr.rest, weight=pr.weight)
    return o


def _gpu(pr, P):
    from paper_1305_3976_b200 import ibgm
    if P == 1:
        return ibgm.from_problem(pr)
    return ibgm.from_problem(pr, nranks=P, transport=EMU)


@pytest.mark.parametrize("dim,n,P", [(3, 32, 2), (3, 32, 4), (3, 32, 8), (3, 32, 16), (3, 128, 8),
                                     (2, 64, 2), (2, 64, 8), (2, 64, 32), (2, 1024, 8), (3, 48, 8)])
@pytest.mark.parametrize("which", ["visc", "psi"])
def test_slab_cut_axis_line_solve(dim, n, P, which):
    """a13: the cross-slab Schur solve along the cut axis vs the oracle's long-double
    Thomas + Sherman-Morrison on identical right-hand sides: <= 1e-12."""
    from oracle import oracle as O
    from paper_1305_3976_b200 import ibgm
    ctx = ibgm.Context(dim, n, 0.01, 1.0, 1e-3, nranks=P, transport=EMU)
    kap = 0.0524 if which == "visc" else float(n) ** 2
    d = RNG.standard_normal((n,) * dim)
    x = ctx.line_solve(dim - 1, kap, d)
    ref = O.solve_axis(d, dim - 1, -kap, 1 + 2 * kap, -kap)
    assert _rel(x, ref) <= 1e-12, _rel(x, ref)
    ctx.close()


def test_slab_cut_axis_line_solve_384_sampled():
    """Config-4 shape over 8 slabs (48 planes each): 64 sampled z-lines per system."""
    from oracle import oracle as O
    from paper_1305_3976_b200 import ibgm
    n = 384
    ctx = ibgm.Context(3, n, 0.005, 1.0, 5e-5, nranks=8, transport=EMU)
    d = RNG.standard_normal((n, n, n))
    for kap in (0.0184, float(n) ** 2):
        x = ctx.line_solve(2, kap, d)
        for _ in range(64):
            a, b = RNG.integers(0, n, 2)
            ref = O.cyclic_solve(-kap, 1 + 2 * kap, -kap, d[:, a, b])
            assert _rel(x[:, a, b], ref) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("cfg,over,P", [(0, {}, 2), (0, {}, 8), (1, dict(n=64, pts=256), 4),
                                        (2, dict(n=128, pts=512), 8), (3, dict(n=32, nodes=2000), 2),
                                        (3, dict(n=32, nodes=2000), 8), (3, dict(n=32, nodes=2000), 16),
                                        (4, dict(n=48, nodes=1500), 8)])
def test_slab_one_step_stages(cfg, over, P):
    """After one step on P slabs: X^{n+1/2}, F, the spread f (owner-only spreading),
    N(u^n) (halo-fed stencils), then u, p, psi, X against the oracle."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(cfg, **over)
    o = _oracle_for(pr)
    g = _gpu(pr, P)
    g.set_debug(True, 0)
    o.step(1)
    g.step(1)
    ao, ag = o.aux(), g.aux()
    assert _rel(ag["Xh"], ao["Xh"]) <= 1e-14
    assert _rel(ag["F"], ao["F"]) <= 1e-12
    for c in range(pr.dim):
        assert _rel(ag["f"][c], ao["f"][c]) <= 1e-12, ("f", c)
        if np.abs(ao["nadv"][c]).max() > 0:
            assert _rel(ag["nadv"][c], ao["nadv"][c]) <= 1e-12, ("N", c)
    fo, fg = o.fields(), g.fields()
    for c in range(pr.dim):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-11, ("u", c)
    assert _rel(fg["p"], fo["p"]) <= 1e-11
    assert _rel(fg["psi"], fo["psi"]) <= 1e-11
    assert _rel(fg["X"], fo["X"]) <= 1e-14
    g.close()


@pytest.mark.parametrize("cfg,over,P", [(0, {}, 4), (1, {}, 8), (2, {}, 8), (3, {}, 8), (3, {}, 2),
                                        (4, dict(n=96, nodes=4000), 8), (4, dict(n=96, nodes=4000), 4)])
def test_slab_ten_step_parity(cfg, over, P):
    """The north_star bar on the decomposition: rel L_inf <= 1e-9 on u, p, X, U after
    10 steps vs the oracle, and <= 1e-10 vs the single-GPU path."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(cfg, **over)
    o = _oracle_for(pr)
    g = _gpu(pr, P)
    g1 = _gpu(pr, 1)
    o.step(10)
    g.step(10)
    g1.step(10)
    fo, fg, f1 = o.fields(), g.fields(), g1.fields()
    for c in range(pr.dim):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9, ("u", c)
        assert _rel(fg["u"][c], f1["u"][c]) <= 1e-10, ("u vs 1 GPU", c)
    assert _rel(fg["p"], fo["p"]) <= 1e-9
    assert _rel(fg["p"], f1["p"]) <= 1e-10
    assert _rel(fg["X"], fo["X"]) <= 1e-9
    assert _rel(fg["X"], f1["X"]) <= 1e-10
    assert _rel(fg["U"], fo["U"]) <= 1e-9
    g.check_finite()
    g.close()
    g1.close()


def test_slab_minimum_depth_and_no_points():
    """nz = 2 (the smallest slab: interior block of one unknown), and a pure fluid."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(1, n=32, pts=64)
    for P, drop in ((16, False), (4, True)):
        if drop:
            pr.X = None
        o = _oracle_for(pr)
        g = _gpu(pr, P)
        o.step(5)
        g.step(5)
        fo, fg = o.fields(), g.fields()
        assert _rel(fg["u"][0], fo["u"][0]) <= 1e-10 and _rel(fg["p"], fo["p"]) <= 1e-10
        g.close()


def test_slab_rejects_bad_decompositions():
    from paper_1305_3976_b200 import ibgm
    for n, P in ((32, 3), (32, 32)):
        with pytest.raises(ibgm.IBGMError) as e:
            ibgm.Context(3, n, 0.01, 1.0, 1e-3, nranks=P, transport=EMU)
        assert e.value.code == -1
    with pytest.raises(ibgm.IBGMError) as e:   # NCCL transport without an id
        ibgm.Context(3, 32, 0.01, 1.0, 1e-3, nranks=2, rank=0)
    assert e.value.code == -1


def test_nccl_unique_id_loads_on_the_gpu_box():
    from paper_1305_3976_b200 import ibgm
    a, b = ibgm.nccl_unique_id(), ibgm.nccl_unique_id()
    assert len(a) == 128 and a != b


@pytest.mark.parametrize("transport", ["nccl", "emulate"])
def test_one_slab_transports(transport):
    """One slab through the slab code path: the NCCL transport on a 1-rank communicator
    (self send/recv carries the periodic halo; all-gather/all-reduce of size 1, captured
    in the step's CUDA graph) and EMULATE with P = 1; both vs the oracle and the
    single-GPU path."""
    from paper_1305_3976_b200 import ibgm, inputs
    pr = inputs.config(3, n=32, nodes=2000)
    if transport == "nccl":
        g = ibgm.from_problem(pr, nranks=1, rank=0, nccl_id=ibgm.nccl_unique_id())
    else:
        g = ibgm.from_problem(pr, nranks=1, transport=EMU)
    g1 = _gpu(pr, 1)
    o = _oracle_for(pr)
    o.step(10); g.step(10); g1.step(10)
    fo, fg, f1 = o.fields(), g.fields(), g1.fields()
    for c in range(3):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9
        assert _rel(fg["u"][c], f1["u"][c]) <= 1e-10
    assert _rel(fg["p"], fo["p"]) <= 1e-9 and _rel(fg["X"], fo["X"]) <= 1e-9
    d = RNG.standard_normal((32, 32, 32))
    x = g.line_solve(2, 32.0 ** 2, d)
    from oracle import oracle as O
    assert _rel(x, O.solve_axis(d, 2, -1024.0, 2049.0, -1024.0)) <= 1e-12
    g.close(); g1.close()


def test_ellipse_array_points_cross_slabs():
    """§8(f4): the 2 x 2 ellipse array of PAPER.md:1972-2003 (box [0,2]^2, background
    velocity (1, sqrt 3)/2) on 4 y-slabs: the membranes drift across slab boundaries
    (replicated Lagrangian data, owner-only spreading, partial interpolation); 30
    steps against the oracle and the single-GPU path."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.ellipse_array(2, n_cell=32, dt_over_h=0.01)
    o = _oracle_for(pr)
    g = _gpu(pr, 4)
    g1 = _gpu(pr, 1)
    o.step(30); g.step(30); g1.step(30)
    fo, fg, f1 = o.fields(), g.fields(), g1.fields()
    for c in range(2):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9 and _rel(fg["u"][c], f1["u"][c]) <= 1e-10
    assert _rel(fg["p"], fo["p"]) <= 1e-9 and _rel(fg["X"], fo["X"]) <= 1e-9
    # the background flow carried the membranes by ~30 dt |u| = 0.3 h
    assert np.abs(fg["X"] - pr.X).max() > 0.1 / 32
    g.close(); g1.close()


@pytest.mark.slow
def test_config4_full_size_eight_slabs_matches_single_gpu():
    """Config 4 at full size (384^3, 8 x 100k-node shells, the 8-GPU workload of
    BASELINE.json) cut into 8 z-slabs of 48 planes (EMULATE): 10 steps equal the
    single-GPU path to 1e-10 (the oracle's full-size check is the single-GPU one,
    test_config4_full_size_one_step)."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(4)
    g1 = _gpu(pr, 1)
    g1.step(10)
    f1 = g1.fields()
    g1.close()
    g = _gpu(pr, 8)
    g.step(10)
    fg = g.fields()
    g.close()
    for c in range(3):
        assert _rel(fg["u"][c], f1["u"][c]) <= 1e-10, c
    assert _rel(fg["p"], f1["p"]) <= 1e-10 and _rel(fg["X"], f1["X"]) <= 1e-10


_DIVN_CASE = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1305_3976_b200 import ibgm, inputs
from oracle import oracle as O
pr = inputs.config(4, n=96, nodes=4000)
o = O.Oracle(pr.dim, pr.n, pr.mu, pr.rho, pr.dt, chi=pr.chi, kernel=pr.kernel, H=pr.H)
o.set_fields(*pr.u, p=pr.p)
o.set_boundary(pr.X, pr.edges, pr.kappa, rest=pr.rest, weight=pr.weight)
o.step(10)
fo = o.fields()
rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
for P in (1, 4):
    g = ibgm.from_problem(pr) if P == 1 else ibgm.from_problem(pr, nranks=P, transport=1)
    g.step(10)
    fg = g.fields()
    g.close()
    errs = [rel(fg["u"][c], fo["u"][c]) for c in range(3)] + [rel(fg["p"], fo["p"]), rel(fg["X"], fo["X"])]
    print(P, errs)
    assert max(errs) <= 1e-9, (P, errs)
"""


def test_divn_handoff_forced_on_a_small_grid():
    """S1 hands D.u^n to the first psi pass (single GPU: k_lines fill; slabs: the cut-axis
    forward phase) only at N >= 256 by default; IBGM_DIVN=1 forces it on config 4 at
    N = 96 in a fresh process: 10 steps vs the oracle on one GPU and on 4 slabs."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _DIVN_CASE.format(root=root)], capture_output=True, text=True,
                       env=dict(os.environ, IBGM_DIVN="1"), timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("cfg,over,P", [(3, dict(n=32, nodes=2000), 4), (0, {}, 2)])
def test_slab_set_fields_after_steps(cfg, over, P):
    """On z-slabs the u halos for the next step's S1 are exchanged during the previous
    step's psi passes (replayed graphs rely on them); ib_set_fields must make the next
    step exchange them again.  step 5, set_fields(new u, p), step 5 vs the oracle."""
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(cfg, **over)
    o = _oracle_for(pr)
    g = _gpu(pr, P)
    o.step(5)
    g.step(5)
    rng = np.random.default_rng(12)
    shp = (pr.n,) * pr.dim
    u2 = [0.05 * rng.standard_normal(shp) for _ in range(pr.dim)]
    p2 = 0.1 * rng.standard_normal(shp)
    if pr.dim == 3:
        o.set_fields(*u2, p=p2)
        g.set_fields(*u2, p=p2)
    else:
        o.set_fields(u2[0], u2[1], None, p2)
        g.set_fields(u2[0], u2[1], None, p2)
    o.step(5)
    g.step(5)
    fo, fg = o.fields(), g.fields()
    for c in range(pr.dim):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9, c
    assert _rel(fg["p"], fo["p"]) <= 1e-9
    assert _rel(fg["X"], fo["X"]) <= 1e-9
    g.close()

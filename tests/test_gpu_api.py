"""GPU tests of the C-ABI's state handling and error surface (include/ibgm.h, SURVEY.md
§8(b)): restarting with ib_set_fields after steps, checkpoint/resume, the sticky
device-raised faults (IB_EDEGENERATE, IB_ENONFINITE, IB_EDOMAIN), ms_per_phase, and the
full-size parity of the quad-lane interpolation in 3D (a block-boundary race would
show only there)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("cfg,over", [(0, {}), (3, dict(n=32, nodes=2000))])
def test_set_fields_after_steps_restarts_from_current_membrane(cfg, over):
    """step 5, ib_set_fields(new u, p), step 5 -- the oracle does the same sequence
    (orc_set_fields keeps X^n and restarts the start-up rules).  The
    look-ahead has already moved the device membrane to X^{n+1}; set_fields must undo it."""
    from paper_1305_3976_b200 import ibgm, inputs
    pr = inputs.config(cfg, **over)
    o = _oracle_for(pr)
    g = ibgm.from_problem(pr)
    o.step(5)
    g.step(5)
    rng = np.random.default_rng(11)
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
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9, ("u", c, _rel(fg["u"][c], fo["u"][c]))
    assert _rel(fg["p"], fo["p"]) <= 1e-9
    assert _rel(fg["X"], fo["X"]) <= 1e-9, _rel(fg["X"], fo["X"])
    assert _rel(fg["U"], fo["U"]) <= 1e-9
    g.close()


@pytest.mark.parametrize("cfg,over", [(0, {}), (3, dict(n=32, nodes=2000))])
def test_checkpoint_resume_continues_exactly(cfg, over):
    """ib_get_state after 7 steps (look-ahead state included), ib_set_state into a fresh
    context with the same boundary, 5 more steps: the same result as 12 uninterrupted
    steps (spreading atomics aside, ~1e-15) and as the oracle's 12 steps (1e-9)."""
    from paper_1305_3976_b200 import ibgm, inputs
    pr = inputs.config(cfg, **over)
    a = ibgm.from_problem(pr)
    a.step(7)
    blob = a.get_state()
    assert blob.nbytes == a.state_size()
    a.step(5)
    fa = a.fields()
    b = ibgm.from_problem(pr)
    b.set_state(blob)
    assert b.stats()["steps"] == 7
    b.step(5)
    fb = b.fields()
    for c in range(pr.dim):
        assert _rel(fb["u"][c], fa["u"][c]) <= 1e-13
    assert _rel(fb["p"], fa["p"]) <= 1e-13 and _rel(fb["X"], fa["X"]) <= 1e-14
    o = _oracle_for(pr)
    o.step(12)
    fo = o.fields()
    for c in range(pr.dim):
        assert _rel(fb["u"][c], fo["u"][c]) <= 1e-9
    assert _rel(fb["p"], fo["p"]) <= 1e-9 and _rel(fb["X"], fo["X"]) <= 1e-9
    # a blob is refused by a context with another boundary or grid
    c2 = ibgm.Context(pr.dim, pr.n * 2, pr.mu / pr.rho, pr.rho, pr.dt, kernel=pr.kernel)
    with pytest.raises(ibgm.IBGMError) as e:
        c2.set_state(blob)
    assert e.value.code == ibgm.IB_EINVAL
    for ctx in (a, b, c2):
        ctx.close()


def test_degenerate_connection_raises():
    """A connection with rest length L != 0 whose endpoints coincide:
    ib_sync / ib_step return IB_EDEGENERATE instead of spreading NaN; ib_set_fields
    clears the fault."""
    from paper_1305_3976_b200 import ibgm
    n = 32
    ctx = ibgm.Context(2, n, 0.01, 1.0, 1e-3)
    ctx.set_fields(np.zeros((n, n)), np.zeros((n, n)))
    X = np.array([[0.5, 0.5], [0.5, 0.5], [0.6, 0.5]])
    ctx.set_boundary(X, [[0, 1], [1, 2]], 10.0, rest=[0.01, 0.0])
    with pytest.raises(ibgm.IBGMError) as e:
        ctx.step(1)     # raised by this call if the force kernel already ran, else by sync
        ctx.sync()
    assert e.value.code == ibgm.IB_EDEGENERATE
    with pytest.raises(ibgm.IBGMError) as e:
        ctx.step(1)     # sticky
    assert e.value.code == ibgm.IB_EDEGENERATE
    f = ctx.fields()
    assert np.isfinite(f["u"][0]).all() and np.isfinite(f["p"]).all()
    # without the rest length the same geometry is fine
    ctx.set_boundary(X, [[0, 1], [1, 2]], 10.0)
    ctx.set_fields(np.zeros((n, n)), np.zeros((n, n)))
    ctx.step(2)
    ctx.sync()
    ctx.close()


def test_in_step_nonfinite_check():
    """The periodic in-step check (ib_set_check_interval) raises IB_ENONFINITE from
    ib_sync after a NaN entered u; interval 0 turns it off."""
    from paper_1305_3976_b200 import ibgm
    n = 16
    for every, expect in ((1, ibgm.IB_ENONFINITE), (0, None)):
        ctx = ibgm.Context(2, n, 0.01, 1.0, 1e-3)
        ctx.set_check_interval(every)
        u = np.zeros((n, n))
        u[3, 4] = np.nan
        ctx.set_fields(u, np.zeros((n, n)))
        if expect is None:
            ctx.step(2)
            ctx.sync()
        else:
            with pytest.raises(ibgm.IBGMError) as e:
                ctx.step(2)
                ctx.sync()
            assert e.value.code == expect
        ctx.close()


def test_point_moving_more_than_a_cell_is_edomain():
    """u = 50 on a 32^2 grid with dt = 1e-3 moves a point 0.05 > h = 1/32 per step:
    IB_EDOMAIN from the in-step check."""
    from paper_1305_3976_b200 import ibgm
    n = 32
    ctx = ibgm.Context(2, n, 0.01, 1.0, 1e-3)
    ctx.set_check_interval(1)
    ctx.set_fields(np.full((n, n), 50.0), np.zeros((n, n)))
    ctx.set_boundary(np.array([[0.3, 0.3], [0.31, 0.3], [0.3, 0.31]]), [[0, 1], [1, 2], [2, 0]], 0.0)
    with pytest.raises(ibgm.IBGMError) as e:
        ctx.step(1)
        ctx.sync()
    assert e.value.code == ibgm.IB_EDOMAIN
    ctx.close()


def test_stats_ms_per_phase():
    """ib_get_stats' ms_per_phase: the average per-step device time of each phase timed
    under ib_set_profiling, 0 (absent) for phases that did not run."""
    from paper_1305_3976_b200 import ibgm, inputs
    pr = inputs.config(3, n=32, nodes=2000)
    g = ibgm.from_problem(pr)
    assert g.stats()["ms_per_phase"] == {}
    g.set_profiling(True)
    g.step(3)
    st = g.stats()
    assert st["steps"] == 3 and st["kernel_launches"] > 0
    ms = st["ms_per_phase"]
    for ph in ("interp_evolve", "force", "spread", "s1_rhs_xsweep", "sweep_y", "sweep_z", "div_psi_first",
               "psi_y", "psi_x_p"):
        assert ms[ph] > 0, ph
    g.close()


@pytest.mark.parametrize("interp_mode", [3, 4, 1])
def test_config3_full_size_interp_modes_parity(interp_mode):
    """Config 3 at full size (128^3, 40k points) with each 3D interpolation kernel: the
    quad-lane kernel's 3 component groups of a point sit in one 192-thread block, whose
    barrier orders the X^n reads before the X^{n+1} writes (a straddling group would read
    a half-updated point in a later wave).  Two steps against the oracle."""
    from paper_1305_3976_b200 import ibgm, inputs
    pr = inputs.config(3)
    g = ibgm.from_problem(pr)
    g.set_debug(False, 0, interp_mode)
    g.step(2)
    fg = g.fields()
    g.close()
    o = _oracle_for(pr)
    o.step(2)
    fo = o.fields()
    assert _rel(fg["X"], fo["X"]) <= 1e-12, _rel(fg["X"], fo["X"])
    assert _rel(fg["U"], fo["U"]) <= 1e-9
    for c in range(3):
        assert _rel(fg["u"][c], fo["u"][c]) <= 1e-9

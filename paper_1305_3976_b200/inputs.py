"""Seeded synthetic inputs for the BASELINE.json configurations 0-4.

This module holds NO arithmetic of the IB-GM method: it only builds initial
conditions (fluid velocity on the MAC faces, membrane geometry, force-connection
lists).  Both the CUDA path (tests, bench.py) and the oracle consume it; it
imports neither.  Recipes are stated in DESIGN.md ("Inputs") and follow SURVEY.md
8(c) readings R8, R10, R11, R15, R19.

Array convention: fields are numpy arrays indexed [j][i] (2D) or [k][j][i] (3D),
x fastest, so the flat index is i + N*(j + N*k).  u lives at (i h, (j+1/2) h, ...),
v at ((i+1/2) h, j h, ...), w at (..., k h).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

COS4 = 0      # 4-point cosine delta (BASELINE.json configs)
PESKIN4 = 1   # paper eq. (discretedelta)


@dataclass
class Problem:
    name: str
    dim: int
    n: int
    mu: float
    rho: float
    dt: float
    steps: int
    kernel: int = COS4
    chi: float = 0.6
    H: float = 1.0                # box side (h = H/N)
    u: List[np.ndarray] = field(default_factory=list)     # dim arrays
    p: Optional[np.ndarray] = None
    X: np.ndarray = None          # [npts][dim]
    edges: np.ndarray = None      # [nedges][2] int64
    kappa: np.ndarray = None      # [nedges]
    rest: Optional[np.ndarray] = None
    weight: np.ndarray = None     # [npts]

    @property
    def ncell(self) -> int:
        return self.n ** self.dim

    @property
    def npts(self) -> int:
        return 0 if self.X is None else self.X.shape[0]


# ------------------------------------------------------------------ geometry
def ellipse_fibre(npts: int, center, axes, sigma: float = 1.0):
    """Closed fibre X_k = c + (a cos 2 pi s_k, b sin 2 pi s_k), s_k = k/npts
    (uniform in s: R8).  Returns X, ring edges, kappa = sigma/h_s^2,
    weight = h_s (R9)."""
    s = np.arange(npts, dtype=np.float64) / npts
    X = np.stack([center[0] + axes[0] * np.cos(2 * np.pi * s),
                  center[1] + axes[1] * np.sin(2 * np.pi * s)], axis=1)
    k = np.arange(npts, dtype=np.int64)
    edges = np.stack([k, (k + 1) % npts], axis=1)
    hs = 1.0 / npts
    kappa = np.full(npts, sigma / hs ** 2)
    weight = np.full(npts, hs)
    return X, edges, kappa, weight


def fibonacci_sphere(npts: int) -> np.ndarray:
    """Near-uniform unit-sphere point set (R11)."""
    i = np.arange(npts, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / npts
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    golden = np.pi * (3.0 - np.sqrt(5.0))
    th = golden * i
    return np.stack([r * np.cos(th), r * np.sin(th), z], axis=1)


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniform random 3x3 rotation from a seeded generator (QR of a Gaussian matrix)."""
    A = rng.standard_normal((3, 3))
    Q, R = np.linalg.qr(A)
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def sphere_triangulation_edges(P: np.ndarray) -> np.ndarray:
    """Unique edges of the convex hull triangulation of points on the unit sphere."""
    from scipy.spatial import ConvexHull
    hull = ConvexHull(P)
    t = hull.simplices.astype(np.int64)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]], axis=0)
    e.sort(axis=1)
    e = np.unique(e, axis=0)
    return e


def ellipsoid_shell(nodes: int, center, axes, rng: np.random.Generator, sigma: float = 1.0):
    """Triangulated ellipsoidal shell (R10, R11): Fibonacci sphere, seeded random
    rotation, convex-hull edges, scaled to the semi-axes.  Edge springs kappa = sigma,
    rest length 0, nodal weight 1."""
    P = fibonacci_sphere(nodes) @ random_rotation(rng).T
    edges = sphere_triangulation_edges(P)
    X = np.asarray(center, np.float64)[None, :] + P * np.asarray(axes, np.float64)[None, :]
    kappa = np.full(edges.shape[0], float(sigma))
    weight = np.ones(nodes)
    return X, edges, kappa, weight


def _nonoverlapping_centres(rng, count, lo, hi, dim, radius, margin, max_tries=100000):
    """Rejection-sample `count` centres in [lo,hi]^dim with |c_i - c_j| > r_i + r_j + margin (R19)."""
    cs: list = []
    tries = 0
    while len(cs) < count:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("could not place non-overlapping bodies")
        c = rng.uniform(lo, hi, size=dim)
        if all(np.linalg.norm(c - cj) > radius[len(cs)] + radius[j] + margin for j, cj in enumerate(cs)):
            cs.append(c)
    return np.array(cs)


# ------------------------------------------------------------------ fluid
def _band_limited(rng, shape, K):
    """Real random field with Gaussian Fourier coefficients on integer wavenumbers
    0 < |k| <= K (R15)."""
    n = shape[0]
    dim = len(shape)
    ks = [np.fft.fftfreq(n, 1.0 / n)] * (dim - 1) + [np.fft.rfftfreq(n, 1.0 / n)]
    grids = np.meshgrid(*ks, indexing="ij")
    k2 = sum(g * g for g in grids)
    mask = (k2 > 0) & (k2 <= K * K)
    coef = (rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape)) * mask
    return np.fft.irfftn(coef, s=shape, axes=tuple(range(dim)))


def random_divfree(dim: int, n: int, K: int, amp: float, seed: int):
    """Random discretely divergence-free MAC velocity (R15): the discrete curl of a
    band-limited random potential (2D stream function at cell corners, 3D vector
    potential on cell edges), so the MAC divergence vanishes to rounding; scaled so
    that max_c max|u_c| = amp.  Arrays [j][i] / [k][j][i]."""
    rng = np.random.default_rng(seed)
    h = 1.0 / n
    shape = (n,) * dim
    # forward difference along grid axis a of a [.., j, i] array: axis index = dim-1-a
    def fd(q, a):
        ax = dim - 1 - a
        return (np.roll(q, -1, axis=ax) - q) / h
    if dim == 2:
        A = _band_limited(rng, shape, K)
        u = [fd(A, 1), -fd(A, 0)]
    else:
        Ax, Ay, Az = (_band_limited(rng, shape, K) for _ in range(3))
        u = [fd(Az, 1) - fd(Ay, 2), fd(Ax, 2) - fd(Az, 0), fd(Ay, 0) - fd(Ax, 1)]
    m = max(np.abs(c).max() for c in u)
    return [np.ascontiguousarray(c * (amp / m)) for c in u]


# ------------------------------------------------------------------ the paper's own problems
# (validation and timing workloads of PAPER.md section 5)
def thin_ellipse(n: int, sigma: float = 1.0, dt: float = 0.04 / 512, mu: float = 0.01) -> Problem:
    """Thin ellipse of PAPER.md:1294-1345: r1 = 5/28, r2 = 7/20 centred at (1/2, 1/2),
    N_s = 19N/4 points uniform in s, stiffness sigma, rest length 0, fluid at rest,
    mu = 0.01, rho = 1, the paper's delta kernel (eq. discretedelta)."""
    ns = 19 * n // 4
    pr = Problem(f"thin_ellipse_n{n}", 2, n, mu, 1.0, dt, 0, kernel=PESKIN4)
    pr.u = [np.zeros((n, n)), np.zeros((n, n))]
    pr.p = np.zeros((n, n))
    pr.X, pr.edges, pr.kappa, pr.weight = ellipse_fibre(ns, (0.5, 0.5), (5.0 / 28.0, 7.0 / 20.0), sigma)
    return pr


def thick_shell(n: int, mu: float = 0.01, dt: float = 0.08 / 512) -> Problem:
    """Thick elliptical shell of PAPER.md:1588-1634: r1 = 0.2, r2 = 0.25, thickness
    gamma = 0.0625, N_s = 75N/16, N_r = 3N/8 circumferential fibres with stiffness
    sigma(r) = 1 - cos 2 pi r, rest length 0; fibre j at r_j = (j + 1/2)/N_r, weights
    h_s h_r (R22); fluid at rest, rho = 1, the paper's delta kernel."""
    ns, nr = 75 * n // 16, 3 * n // 8
    r1, r2, gam = 0.2, 0.25, 0.0625
    s = np.arange(ns) / ns
    Xs, Es, Ks = [], [], []
    for jr in range(nr):
        r = (jr + 0.5) / nr
        Xs.append(np.stack([0.5 + (r1 + gam * (r - 0.5)) * np.cos(2 * np.pi * s),
                            0.5 + (r2 + gam * (r - 0.5)) * np.sin(2 * np.pi * s)], 1))
        k = np.arange(ns)
        Es.append(np.stack([k, (k + 1) % ns], 1) + jr * ns)
        Ks.append(np.full(ns, (1 - np.cos(2 * np.pi * r)) * ns ** 2))
    pr = Problem(f"thick_shell_n{n}", 2, n, mu, 1.0, dt, 0, kernel=PESKIN4)
    pr.u = [np.zeros((n, n)), np.zeros((n, n))]
    pr.p = np.zeros((n, n))
    pr.X = np.ascontiguousarray(np.concatenate(Xs))
    pr.edges = np.ascontiguousarray(np.concatenate(Es).astype(np.int64))
    pr.kappa = np.concatenate(Ks)
    pr.weight = np.full(ns * nr, 1.0 / (ns * nr))
    return pr


def cylinder_shell(n: int, sigma_s: float = 1.0, sigma_r: float = 1.0, rest: float = 1.0,
                   mu: float = 0.01) -> Problem:
    """3D cylindrical shell of PAPER.md:2078-2118: X(s, r) = (r, 1/2 + r1 cos 2 pi s,
    1/2 + r2 sin 2 pi s), r1 = 5/28, r2 = 7/20, N_s = 19N/4 fibres around (stiffness
    sigma_s, rest length 0) interwoven with N_r = 3N axial fibres (stiffness sigma_r,
    rest length L = 1), periodic in x (no cuts), dt = 0.04/N.  Force connections in the
    form of PAPER.md:856-861: kappa = sigma/h^2 and rest length L h along each family,
    quadrature weight h_s h_r (R26)."""
    ns, nr = 19 * n // 4, 3 * n
    hs, hr = 1.0 / ns, 1.0 / nr
    r1, r2 = 5.0 / 28.0, 7.0 / 20.0
    s = np.arange(ns) / ns
    r = np.arange(nr) / nr
    R, S = np.meshgrid(r, s, indexing="ij")            # point (jr, js) -> jr * ns + js
    X = np.stack([R.ravel(), (0.5 + r1 * np.cos(2 * np.pi * S)).ravel(),
                  (0.5 + r2 * np.sin(2 * np.pi * S)).ravel()], 1)
    jr, js = np.meshgrid(np.arange(nr), np.arange(ns), indexing="ij")
    idx = jr * ns + js
    e_s = np.stack([idx.ravel(), (jr * ns + (js + 1) % ns).ravel()], 1)
    e_r = np.stack([idx.ravel(), (((jr + 1) % nr) * ns + js).ravel()], 1)
    pr = Problem(f"cylinder_n{n}", 3, n, mu, 1.0, 0.04 / n, 100, kernel=PESKIN4)
    pr.u = [np.zeros((n, n, n)) for _ in range(3)]
    pr.p = np.zeros((n, n, n))
    pr.X = np.ascontiguousarray(X)
    pr.edges = np.ascontiguousarray(np.concatenate([e_s, e_r]).astype(np.int64))
    pr.kappa = np.concatenate([np.full(len(e_s), sigma_s / hs ** 2), np.full(len(e_r), sigma_r / hr ** 2)])
    pr.rest = np.concatenate([np.zeros(len(e_s)), np.full(len(e_r), rest * hr)])
    pr.weight = np.full(ns * nr, hs * hr)
    return pr


def ellipse_array(P: int, n_cell: int = 128, sigma: float = 1.0, t_background=(0.5, 0.5 * np.sqrt(3.0)),
                  dt_over_h: float = 0.01, mu: float = 0.01) -> Problem:
    """P x P array of thin ellipses of PAPER.md:1972-2003 on the box [0, P]^2 (H = P,
    N = P n_cell, h = 1/n_cell): ellipse (l, m) centred in its unit cell, r1 = 5/28,
    r2 = 7/20, h_s = 4h/19 (N_s = 19 n_cell/4 points), sigma = 1, constant background
    velocity u(x, 0) = (1, sqrt 3)/2, dt = 0.01 h, the paper's delta kernel."""
    n = P * n_cell
    h = 1.0 / n_cell
    ns = 19 * n_cell // 4
    pr = Problem(f"ellipse_array_{P}x{P}_n{n_cell}", 2, n, mu, 1.0, dt_over_h * h, 0, kernel=PESKIN4, H=float(P))
    pr.u = [np.full((n, n), float(t_background[0])), np.full((n, n), float(t_background[1]))]
    pr.p = np.zeros((n, n))
    parts = [ellipse_fibre(ns, (l + 0.5, m + 0.5), (5.0 / 28.0, 7.0 / 20.0), sigma)
             for m in range(P) for l in range(P)]
    pr.X, pr.edges, pr.kappa, pr.weight = _concat(parts)
    return pr


# ------------------------------------------------------------------ configs
def config(idx: int, **over) -> Problem:
    """BASELINE.json configs[idx]; keyword overrides (n=, nodes=, pts=, steps=) give
    scaled-down variants for tests.  Seeds: 13051.. (DESIGN.md Inputs)."""
    if idx == 0:
        n = over.get("n", 32)
        pts = over.get("pts", 128)
        pr = Problem("cfg0", 2, n, 0.01, 1.0, over.get("dt", 1e-3), over.get("steps", 20))
        pr.u = [np.zeros((n, n)), np.zeros((n, n))]
        pr.X, pr.edges, pr.kappa, pr.weight = ellipse_fibre(pts, (0.5, 0.5), (0.2, 0.15))
    elif idx == 1:
        n = over.get("n", 256)
        pts = over.get("pts", 1024)
        pr = Problem("cfg1", 2, n, 0.01, 1.0, over.get("dt", 1e-4), over.get("steps", 200))
        pr.u = random_divfree(2, n, 8, 0.05, seed=13051)
        pr.X, pr.edges, pr.kappa, pr.weight = ellipse_fibre(pts, (0.5, 0.5), (0.2, 0.15))
    elif idx == 2:
        n = over.get("n", 1024)
        pts = over.get("pts", 2048)
        pr = Problem("cfg2", 2, n, 0.005, 1.0, over.get("dt", 2e-5), over.get("steps", 100))
        pr.u = [np.zeros((n, n)), np.zeros((n, n))]
        rng = np.random.default_rng(13052)
        axes = rng.uniform(0.05, 0.12, size=(4, 2))
        cen = _nonoverlapping_centres(rng, 4, 0.2, 0.8, 2, axes.max(axis=1), 4.0 / n)
        parts = [ellipse_fibre(pts, cen[b], axes[b]) for b in range(4)]
        pr.X, pr.edges, pr.kappa, pr.weight = _concat(parts)
    elif idx == 3:
        n = over.get("n", 128)
        nodes = over.get("nodes", 40000)
        pr = Problem("cfg3", 3, n, 0.01, 1.0, over.get("dt", 1e-4), over.get("steps", 100))
        pr.u = [np.zeros((n, n, n)) for _ in range(3)]
        rng = np.random.default_rng(13053)
        pr.X, pr.edges, pr.kappa, pr.weight = ellipsoid_shell(nodes, (0.5, 0.5, 0.5), (0.2, 0.15, 0.15), rng)
    elif idx == 4:
        n = over.get("n", 384)
        nodes = over.get("nodes", 100000)
        pr = Problem("cfg4", 3, n, 0.005, 1.0, over.get("dt", 5e-5), over.get("steps", 20))
        pr.u = random_divfree(3, n, 6, 0.02, seed=13054)
        rng = np.random.default_rng(13055)
        axes = rng.uniform(0.05, 0.1, size=(8, 3))
        cen = _nonoverlapping_centres(rng, 8, 0.15, 0.85, 3, axes.max(axis=1), 4.0 / n)
        parts = [ellipsoid_shell(nodes, cen[b], axes[b], rng) for b in range(8)]
        pr.X, pr.edges, pr.kappa, pr.weight = _concat(parts)
    else:
        raise ValueError(f"no config {idx}")
    pr.p = np.zeros_like(pr.u[0])
    if "kernel" in over:
        pr.kernel = over["kernel"]
    return pr


def _concat(parts):
    Xs, Es, Ks, Ws = [], [], [], []
    off = 0
    for X, E, K, W in parts:
        Xs.append(X); Es.append(E + off); Ks.append(K); Ws.append(W)
        off += X.shape[0]
    return (np.ascontiguousarray(np.concatenate(Xs)), np.ascontiguousarray(np.concatenate(Es)),
            np.concatenate(Ks), np.concatenate(Ws))

"""ctypes wrapper of the C oracle (oracle/ibgm_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module.  It builds nothing on the product path and shares no code with
paper_1305_3976_b200/.  Argument marshalling only: every number comes from the C.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ibgm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

COS4 = 0
PESKIN4 = 1

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off, plain C99)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-std=gnu99", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        # IBGM_ORACLE_LIB: load a prebuilt variant (tools/oracle_mutants.py builds
        # deliberately broken copies to show each pin fails on them)
        _lib = ctypes.CDLL(os.environ.get("IBGM_ORACLE_LIB") or build())
        L = _lib
        L.orc_phi.restype = ctypes.c_double
        L.orc_phi.argtypes = [ctypes.c_int, ctypes.c_double]
        L.orc_cyclic_solve.argtypes = [ctypes.c_long, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, _dp, _dp]
        L.orc_solve_axis.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, _dp]
        L.orc_op_d2.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_int, _dp, _dp]
        L.orc_op_grad.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_int, _dp, _dp]
        L.orc_op_div.argtypes = [ctypes.c_int, ctypes.c_long, _dp, _dp, _dp, _dp]
        L.orc_op_adv.argtypes = [ctypes.c_int, ctypes.c_long, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_op_interp.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_int, _dp, _dp, _dp,
                                    ctypes.c_long, _dp, _dp]
        L.orc_op_spread.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_int, ctypes.c_long,
                                    _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_op_force.argtypes = [ctypes.c_int, ctypes.c_long, _dp, ctypes.c_long, _i64p,
                                   _dp, _dp, _dp]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int]
        L.orc_create_box.restype = ctypes.c_void_p
        L.orc_create_box.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int]
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_set_fields.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp]
        L.orc_set_boundary.restype = ctypes.c_int
        L.orc_set_boundary.argtypes = [ctypes.c_void_p, ctypes.c_long, _dp, ctypes.c_long, _i64p,
                                       _dp, _dp, _dp]
        L.orc_step.argtypes = [ctypes.c_void_p, ctypes.c_long]
        L.orc_get_fields.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_get_aux.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_keep_ustar.restype = ctypes.c_int
        L.orc_keep_ustar.argtypes = [ctypes.c_void_p]
        L.orc_get_ustar.restype = ctypes.c_int
        L.orc_get_ustar.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp]
        L.orc_steps_done.restype = ctypes.c_long
        L.orc_steps_done.argtypes = [ctypes.c_void_p]
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "oracle wants C-contiguous f64"
    return a.ctypes.data_as(_dp)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- primitives
def phi(kernel: int, r) -> np.ndarray:
    L = lib()
    r = np.atleast_1d(np.asarray(r, dtype=np.float64))
    return np.array([L.orc_phi(kernel, float(x)) for x in r.ravel()]).reshape(r.shape)


def cyclic_solve(c: float, a: float, b: float, d) -> np.ndarray:
    d = _c(d)
    x = np.empty_like(d)
    lib().orc_cyclic_solve(d.size, c, a, b, _p(d), _p(x))
    return x


def solve_axis(q, axis: int, c: float, a: float, b: float) -> np.ndarray:
    """Cyclic solve of every grid line of q along `axis` (0 = x, the last array axis)."""
    q = _c(q).copy()
    lib().orc_solve_axis(q.ndim, q.shape[0], axis, c, a, b, _p(q))
    return q


def _shape(dim, n):
    return (n, n) if dim == 2 else (n, n, n)


def d2(q, axis: int) -> np.ndarray:
    """D_aa q; arrays are indexed [k][j][i] (x fastest)."""
    q = _c(q)
    dim = q.ndim
    out = np.empty_like(q)
    lib().orc_op_d2(dim, q.shape[0], axis, _p(q), _p(out))
    return out


def grad(p, comp: int) -> np.ndarray:
    p = _c(p)
    out = np.empty_like(p)
    lib().orc_op_grad(p.ndim, p.shape[0], comp, _p(p), _p(out))
    return out


def div(u, v, w=None) -> np.ndarray:
    u, v = _c(u), _c(v)
    w = None if w is None else _c(w)
    out = np.empty_like(u)
    lib().orc_op_div(u.ndim, u.shape[0], _p(u), _p(v), _p(w), _p(out))
    return out


def adv(u, v, w=None):
    u, v = _c(u), _c(v)
    w = None if w is None else _c(w)
    nu, nv = np.empty_like(u), np.empty_like(v)
    nw = None if w is None else np.empty_like(w)
    lib().orc_op_adv(u.ndim, u.shape[0], _p(u), _p(v), _p(w), _p(nu), _p(nv), _p(nw))
    return (nu, nv) if w is None else (nu, nv, nw)


def interp(kernel, u, v, w, X) -> np.ndarray:
    u, v = _c(u), _c(v)
    w = None if w is None else _c(w)
    X = _c(X)
    dim = u.ndim
    U = np.empty_like(X)
    lib().orc_op_interp(dim, u.shape[0], kernel, _p(u), _p(v), _p(w), X.shape[0], _p(X), _p(U))
    return U


def spread(kernel, dim, n, X, F, wgt=None):
    X, F = _c(X), _c(F)
    wgt = None if wgt is None else _c(wgt)
    f = [np.zeros(_shape(dim, n)) for _ in range(dim)]
    lib().orc_op_spread(dim, n, kernel, X.shape[0], _p(X), _p(F), _p(wgt), _p(f[0]), _p(f[1]),
                        _p(f[2]) if dim == 3 else None)
    return f


def force(X, edges, kappa, rest=None) -> np.ndarray:
    X = _c(X)
    edges = np.ascontiguousarray(edges, dtype=np.int64)
    kappa = _c(np.broadcast_to(np.asarray(kappa, dtype=np.float64), (edges.shape[0],)))
    rest = None if rest is None else _c(np.broadcast_to(np.asarray(rest, np.float64), (edges.shape[0],)))
    F = np.empty_like(X)
    lib().orc_op_force(X.shape[1], X.shape[0], _p(X), edges.shape[0],
                       edges.ctypes.data_as(_i64p), _p(kappa), _p(rest), _p(F))
    return F


# ---------------------------------------------------------------- full step
class Oracle:
    """Plain CPU IB-GM stepper (the test oracle).  Field arrays are numpy
    [k][j][i] (3D) or [j][i] (2D), x fastest."""

    def __init__(self, dim, n, mu, rho, dt, chi=0.6, kernel=COS4, advection=True, rotate=True, H=1.0):
        self.dim, self.n = dim, n
        self._h = lib().orc_create_box(dim, n, H, mu, rho, dt, chi, kernel, int(advection), int(rotate))
        if not self._h:
            raise MemoryError("orc_create failed")
        self.npts = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_destroy(h)
            self._h = None

    def set_fields(self, u, v, w=None, p=None):
        self._keep = [_c(u), _c(v), None if w is None else _c(w), None if p is None else _c(p)]
        k = self._keep
        lib().orc_set_fields(self._h, _p(k[0]), _p(k[1]), _p(k[2]), _p(k[3]))

    def set_boundary(self, X, edges, kappa, rest=None, weight=None):
        X = _c(X)
        edges = np.ascontiguousarray(edges, dtype=np.int64)
        ne = edges.shape[0]
        kappa = _c(np.broadcast_to(np.asarray(kappa, np.float64), (ne,)))
        rest = None if rest is None else _c(np.broadcast_to(np.asarray(rest, np.float64), (ne,)))
        weight = None if weight is None else _c(np.broadcast_to(np.asarray(weight, np.float64), (X.shape[0],)))
        rc = lib().orc_set_boundary(self._h, X.shape[0], _p(X), ne, edges.ctypes.data_as(_i64p),
                                    _p(kappa), _p(rest), _p(weight))
        if rc != 0:
            raise ValueError("edge index out of range")
        self.npts = X.shape[0]

    def step(self, nsteps=1):
        lib().orc_step(self._h, nsteps)

    @property
    def steps_done(self):
        return lib().orc_steps_done(self._h)

    def fields(self):
        shp = _shape(self.dim, self.n)
        u = [np.empty(shp) for _ in range(self.dim)]
        p, psi = np.empty(shp), np.empty(shp)
        X = np.empty((self.npts, self.dim))
        U = np.empty((self.npts, self.dim))
        lib().orc_get_fields(self._h, _p(u[0]), _p(u[1]), _p(u[2]) if self.dim == 3 else None,
                             _p(p), _p(psi), _p(X) if self.npts else None, _p(U) if self.npts else None)
        return dict(u=u, p=p, psi=psi, X=X, U=U)

    def keep_ustar(self):
        """Test hook: keep u* (Step 3b) and p* (Step 3a) of every following step."""
        if lib().orc_keep_ustar(self._h) != 0:
            raise MemoryError("orc_keep_ustar failed")

    def ustar(self):
        shp = _shape(self.dim, self.n)
        us = [np.empty(shp) for _ in range(self.dim)]
        ps = np.empty(shp)
        rc = lib().orc_get_ustar(self._h, _p(us[0]), _p(us[1]), _p(us[2]) if self.dim == 3 else None, _p(ps))
        if rc != 0:
            raise RuntimeError("call keep_ustar() before stepping")
        return dict(ustar=us, pstar=ps)

    def aux(self):
        shp = _shape(self.dim, self.n)
        f = [np.empty(shp) for _ in range(self.dim)]
        nadv = [np.empty(shp) for _ in range(self.dim)]
        F = np.empty((self.npts, self.dim))
        Xh = np.empty((self.npts, self.dim))
        d3 = self.dim == 3
        lib().orc_get_aux(self._h, _p(f[0]), _p(f[1]), _p(f[2]) if d3 else None,
                          _p(nadv[0]), _p(nadv[1]), _p(nadv[2]) if d3 else None,
                          _p(F) if self.npts else None, _p(Xh) if self.npts else None)
        return dict(f=f, nadv=nadv, F=F, Xh=Xh)

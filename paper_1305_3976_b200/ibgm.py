"""Thin Python binding of libibgm.so (include/ibgm.h).

Argument marshalling only: every step of the method runs in the CUDA kernels of
the library.  There is no CPU fallback: if libibgm.so is missing or cannot be
loaded, importing `lib()` raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

IB_DELTA_COS4 = 0
IB_DELTA_PESKIN4 = 1
IB_TRANSPORT_NCCL = 0
IB_TRANSPORT_EMULATE = 1

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class IBGMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libibgm error {code}: {msg}")
        self.code = code


class ib_grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n", ctypes.c_int64), ("H", ctypes.c_double)]


class ib_options(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("chi", ctypes.c_double), ("advection", ctypes.c_int32),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("transport", ctypes.c_int32), ("nccl_id", ctypes.c_void_p)]


_lib = None
SYMBOLS = ["ib_default_options", "ib_create", "ib_set_fields", "ib_set_boundary", "ib_set_fibers",
           "ib_step", "ib_sync", "ib_get_fields", "ib_get_aux", "ib_line_solve", "ib_check_finite",
           "ib_get_stats", "ib_destroy", "ib_last_error", "ib_set_profiling", "ib_get_phase_times",
           "ib_set_debug", "ib_nccl_unique_id", "ib_slab_range", "ib_psi_solve", "ib_set_check_interval",
           "ib_state_size", "ib_get_state", "ib_set_state"]

IB_OK, IB_EINVAL, IB_ESTATE, IB_ECUDA, IB_ENCCL = 0, -1, -2, -3, -4
IB_ENONFINITE, IB_EDOMAIN, IB_ENOMEM, IB_EDEGENERATE = -5, -6, -7, -8

PHASES = ["interp_evolve", "force", "spread", "s1_rhs_xsweep", "sweep_y", "sweep_z", "div_psi_first",
          "psi_y", "psi_x_p", "clear"]


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load libibgm.so (building it first if sources are newer and nvcc exists)."""
    global _lib
    if _lib is None:
        path = os.environ.get("IBGM_LIB_PATH") or _build.LIB     # dev A/B builds only
        if path == _build.LIB and _build.needs_build():
            try:
                _build.build()
            except Exception as e:  # noqa: BLE001
                if not os.path.exists(path):
                    raise RuntimeError(f"libibgm.so is missing and could not be built: {e}") from e
        L = ctypes.CDLL(path)
        L.ib_default_options.argtypes = [ctypes.POINTER(ib_options)]
        L.ib_create.argtypes = [ctypes.POINTER(ib_grid), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.POINTER(ib_options), ctypes.POINTER(ctypes.c_void_p)]
        L.ib_set_fields.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp]
        L.ib_set_boundary.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp, ctypes.c_int64, _i64p, _dp, _dp, _dp]
        L.ib_set_fibers.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i64p, _dp, ctypes.c_double]
        L.ib_step.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.ib_sync.argtypes = [ctypes.c_void_p]
        L.ib_get_fields.argtypes = [ctypes.c_void_p] + [_dp] * 7
        L.ib_get_aux.argtypes = [ctypes.c_void_p] + [_dp] * 8
        L.ib_line_solve.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, _dp, _dp]
        L.ib_check_finite.argtypes = [ctypes.c_void_p]
        L.ib_get_stats.argtypes = [ctypes.c_void_p, _dp, _i64p, _i64p]
        L.ib_set_check_interval.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.ib_state_size.argtypes = [ctypes.c_void_p, _i64p]
        L.ib_get_state.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.ib_set_state.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.ib_destroy.argtypes = [ctypes.c_void_p]
        L.ib_last_error.restype = ctypes.c_char_p
        L.ib_set_profiling.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.ib_get_phase_times.argtypes = [ctypes.c_void_p, _dp, _i64p]
        L.ib_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.ib_nccl_unique_id.argtypes = [ctypes.c_void_p]
        L.ib_psi_solve.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int32, _dp]
        L.ib_slab_range.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _i64p, _i64p]
        for name in SYMBOLS:
            if name not in ("ib_default_options", "ib_last_error"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _ck(rc):
    if rc != 0:
        raise IBGMError(rc, lib().ib_last_error().decode())


def _p(a):
    if a is None:
        return None
    if not (a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise TypeError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(_dp)


def _c(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def nccl_unique_id() -> bytes:
    """ib_nccl_unique_id: 128 bytes for rank 0 to share with every rank."""
    buf = ctypes.create_string_buffer(128)
    _ck(lib().ib_nccl_unique_id(buf))
    return buf.raw


def slab_range(n, nranks, rank):
    """ib_slab_range: (z0, nz) of rank's slab along the cut axis."""
    z0, nz = ctypes.c_int64(), ctypes.c_int64()
    _ck(lib().ib_slab_range(n, nranks, rank, ctypes.byref(z0), ctypes.byref(nz)))
    return z0.value, nz.value


def share_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it (any backend)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class Context:
    """One IB-GM problem: ib_create(grid, nu, rho, dt).

    nranks > 1 cuts the grid into z-slabs: transport
    IB_TRANSPORT_NCCL holds this rank's slab (fields are local, nccl_id from
    share_nccl_id()), IB_TRANSPORT_EMULATE holds all slabs on one GPU (fields are
    global)."""

    def __init__(self, dim, n, nu, rho, dt, *, kernel=IB_DELTA_COS4, chi=0.6, advection=True, device=0,
                 stream=None, nranks=1, rank=0, transport=IB_TRANSPORT_NCCL, nccl_id=None, H=1.0):
        L = lib()
        self.dim, self.n = dim, n
        self.nranks, self.rank, self.transport = nranks, rank, transport
        self.local = nranks > 1 and transport == IB_TRANSPORT_NCCL   # fields are this rank's slab
        self.nz = n // nranks if self.local else n
        g = ib_grid(dim, n, float(H))
        o = ib_options()
        L.ib_default_options(ctypes.byref(o))
        o.kernel, o.chi, o.advection, o.device = kernel, chi, int(advection), device
        o.stream = stream
        o.nranks, o.rank, o.transport = nranks, rank, transport
        self._id = None
        if nccl_id is not None:
            self._id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._id, ctypes.c_void_p)
        h = ctypes.c_void_p()
        rc = L.ib_create(ctypes.byref(g), nu, rho, dt, ctypes.byref(o), ctypes.byref(h))
        self._h = h
        if rc != 0:
            msg = L.ib_last_error().decode()
            if h.value:
                L.ib_destroy(h)
            self._h = None
            raise IBGMError(rc, msg)
        self.npts = 0

    @property
    def shape(self):
        """Shape of the field arrays this context takes and returns (the local slab with
        the NCCL transport)."""
        return (self.nz,) + (self.n,) * (self.dim - 1)

    def close(self):
        h = getattr(self, "_h", None)
        self._h = None
        L = _lib   # module globals may already be torn down at interpreter exit
        if h and L is not None:
            L.ib_destroy(h)

    def __del__(self):
        self.close()

    def set_fields(self, u, v, w=None, p=None):
        u, v, w, p = _c(u), _c(v), _c(w), _c(p)
        _ck(lib().ib_set_fields(self._h, _p(u), _p(v), _p(w), _p(p)))

    def set_boundary(self, X, edges, kappa, rest=None, weight=None):
        X = _c(X)
        edges = np.ascontiguousarray(edges, dtype=np.int64).reshape(-1, 2)
        ne = edges.shape[0]
        kappa = _c(np.broadcast_to(np.asarray(kappa, np.float64), (ne,)))
        rest = None if rest is None else _c(np.broadcast_to(np.asarray(rest, np.float64), (ne,)))
        npts = 0 if X is None else X.shape[0]
        weight = None if weight is None else _c(np.broadcast_to(np.asarray(weight, np.float64), (npts,)))
        _ck(lib().ib_set_boundary(self._h, npts, _p(X), ne, edges.ctypes.data_as(_i64p), _p(kappa), _p(rest),
                                  _p(weight)))
        self.npts = npts

    def set_fibers(self, pts_per_fiber, X, sigma):
        X = _c(X)
        ppf = np.ascontiguousarray(pts_per_fiber, dtype=np.int64)
        _ck(lib().ib_set_fibers(self._h, len(ppf), ppf.ctypes.data_as(_i64p), _p(X), sigma))
        self.npts = X.shape[0]

    def step(self, nsteps=1):
        _ck(lib().ib_step(self._h, nsteps))

    def sync(self):
        _ck(lib().ib_sync(self._h))

    def fields(self):
        u = [np.empty(self.shape) for _ in range(self.dim)]
        p, psi = np.empty(self.shape), np.empty(self.shape)
        X = np.empty((self.npts, self.dim))
        U = np.empty((self.npts, self.dim))
        _ck(lib().ib_get_fields(self._h, _p(u[0]), _p(u[1]), _p(u[2]) if self.dim == 3 else None, _p(p), _p(psi),
                                _p(X) if self.npts else None, _p(U) if self.npts else None))
        return dict(u=u, p=p, psi=psi, X=X, U=U)

    def positions(self):
        """X^n only ([npts][dim], caller's point order)."""
        X = np.empty((self.npts, self.dim))
        if self.npts:
            _ck(lib().ib_get_fields(self._h, None, None, None, None, None, _p(X), None))
        return X

    def get_fields_into(self, u, v, w, p, X):
        """D2H into caller buffers (e.g. pinned); any may be None."""
        _ck(lib().ib_get_fields(self._h, _p(u), _p(v), _p(w), _p(p), None, _p(X), None))

    def aux(self, with_f=True):
        d3 = self.dim == 3
        f = [np.empty(self.shape) for _ in range(self.dim)] if with_f else [None] * 3
        nadv = [np.empty(self.shape) for _ in range(self.dim)]
        F = np.empty((self.npts, self.dim))
        Xh = np.empty((self.npts, self.dim))
        _ck(lib().ib_get_aux(self._h, _p(f[0]), _p(f[1]), _p(f[2]) if d3 else None, _p(nadv[0]), _p(nadv[1]),
                             _p(nadv[2]) if d3 else None, _p(F) if self.npts else None,
                             _p(Xh) if self.npts else None))
        return dict(f=f, nadv=nadv, F=F, Xh=Xh)

    def line_solve(self, axis, kappa, d):
        d = _c(d)
        x = np.empty_like(d)
        _ck(lib().ib_line_solve(self._h, axis, kappa, _p(d), _p(x)))
        return x

    def psi_solve(self, f, repeats=1):
        """ib_psi_solve: A^{-repeats} f with A = prod_a (1 - D_aa); returns (psi, device ms
        per application)."""
        f = _c(f)
        x = np.empty_like(f)
        ms = ctypes.c_double()
        _ck(lib().ib_psi_solve(self._h, _p(f), _p(x), int(repeats), ctypes.byref(ms)))
        return x, ms.value

    def check_finite(self):
        _ck(lib().ib_check_finite(self._h))

    def set_debug(self, keep_f: bool, spread_mode: int = 0, interp_mode: int = 0):
        """keep_f: keep f^{n+1/2} for aux(); spread_mode: 0 auto, 1 per-point, 2 brick-binned,
        3 box-staged, 4 quad-lane, 5 quad-lane with warp pre-reduction, 6 window-staged;
        interp_mode: 0 auto, 1 per-point, 2 box-staged, 3 quad-lane, 4 per (point, component),
        5 window-staged."""
        _ck(lib().ib_set_debug(self._h, int(keep_f) | (int(spread_mode) << 1) | (int(interp_mode) << 4)))

    def set_profiling(self, on: bool):
        _ck(lib().ib_set_profiling(self._h, int(on)))

    def phase_times(self):
        ms = np.zeros(len(PHASES))
        cnt = np.zeros(len(PHASES), dtype=np.int64)
        _ck(lib().ib_get_phase_times(self._h, _p(ms), cnt.ctypes.data_as(_i64p)))
        return {PHASES[i]: (float(ms[i]), int(cnt[i])) for i in range(len(PHASES)) if cnt[i] > 0}

    def stats(self):
        ms = np.zeros(len(PHASES))
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _ck(lib().ib_get_stats(self._h, _p(ms), ctypes.byref(b), ctypes.byref(a)))
        return dict(kernel_launches=a.value, steps=b.value,
                    ms_per_phase={PHASES[i]: float(ms[i]) for i in range(len(PHASES)) if ms[i] > 0})

    def set_check_interval(self, every: int):
        _ck(lib().ib_set_check_interval(self._h, int(every)))

    def state_size(self) -> int:
        n = ctypes.c_int64()
        _ck(lib().ib_state_size(self._h, ctypes.byref(n)))
        return n.value

    def get_state(self, buf=None):
        """ib_get_state into `buf` (a writable uint8 buffer, e.g. pinned; allocated if None)."""
        n = self.state_size()
        if buf is None:
            buf = np.empty(n, dtype=np.uint8)
        if buf.nbytes < n or not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("state buffer too small or not contiguous")
        _ck(lib().ib_get_state(self._h, ctypes.c_void_p(buf.ctypes.data), buf.nbytes))
        return buf

    def set_state(self, buf):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("state buffer must be contiguous")
        _ck(lib().ib_set_state(self._h, ctypes.c_void_p(buf.ctypes.data), buf.nbytes))


def slab_of(a, nranks, rank):
    """The planes of rank's slab of a global field (cut along the first array axis =
    the last grid axis)."""
    nz = a.shape[0] // nranks
    return np.ascontiguousarray(a[rank * nz:(rank + 1) * nz])


def from_problem(pr, **kw):
    """Context + state from an inputs.Problem (fields cut to the local slab when the
    context holds one)."""
    ctx = Context(pr.dim, pr.n, pr.mu / pr.rho, pr.rho, pr.dt, kernel=pr.kernel, chi=pr.chi, H=pr.H, **kw)
    cut = (lambda a: a if a is None or not ctx.local else slab_of(a, ctx.nranks, ctx.rank))
    u = [cut(x) for x in pr.u]
    p = cut(pr.p)
    ctx.set_fields(*u, p=p) if pr.dim == 3 else ctx.set_fields(u[0], u[1], None, p)
    if pr.X is not None:
        ctx.set_boundary(pr.X, pr.edges, pr.kappa, rest=pr.rest, weight=pr.weight)
    return ctx

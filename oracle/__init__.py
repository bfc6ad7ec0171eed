"""CPU oracle for the wind-downscaling hot path -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liborc.so`` (plain C, fp64, ``-ffp-contract=off``; built by
``__graft_entry__.build()`` / ``make oracle``) and wraps it for numpy arrays.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package; the
product package ``paper_2101_08453_b200`` never does.

Every wrapped function cites the passage of /root/reference/PAPER.md it
follows in ``oracle/orc.c``.  Storage: node arrays (n3, n2, n1); element
arrays (3, nz, ny, nx); K full 27-point, shape (n3, n2, n1, 27) with
o = (dx+1) + 3(dy+1) + 9(dz+1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liborc.so")

RULES = {"coupling_cur": 0, "coupling_paper": 1, "verbatim": 2, "full": 3}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(force=False):
    src = os.path.join(_HERE, "orc.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-std=c11",
                               "-shared", "-fPIC", "-o", _LIB, src, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_mg_setup.restype = C.c_void_p
        L.orc_mg_setup.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                   _ip]
        L.orc_mg_free.argtypes = [C.c_void_p]
        L.orc_mg_K.restype = _dp
        L.orc_mg_K.argtypes = [C.c_void_p, C.c_int]
        for name in ("orc_mg_nlevels", "orc_mg_coarse_direct"):
            getattr(L, name).argtypes = [C.c_void_p]
        L.orc_mg_level_dims.argtypes = [C.c_void_p, C.c_int, _ip]
        L.orc_mg_plan.argtypes = [C.c_void_p, C.c_int, _ip, _ip]
        for name in ("orc_mg_gs", "orc_mg_apply", "orc_mg_restrict", "orc_mg_prolong"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.orc_mg_coarse_solve.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_mg_set_smoother.argtypes = [C.c_void_p, C.c_int]
        L.orc_mg_vcycle.argtypes = [C.c_void_p, _dp, _dp]
        L.orc_mg_solve.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, _dp, _dp, _ip, _dp]
        L.orc_validate_mesh.restype = C.c_longlong
        L.orc_build_mesh.restype = C.c_longlong
        L.orc_build_mesh.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_double, _dp, C.c_int, C.c_double, _dp, _dp, _dp]
        L.orc_interp_wind.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_double, C.c_double, _dp, _dp, _dp, _dp, C.c_int, C.c_int,
                                      C.c_int, _dp]
        L.orc_residual.restype = C.c_double
        L.orc_norm2.restype = C.c_double
        L.orc_plan_level.argtypes = [C.c_double, _dp, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_int, C.c_int, C.c_int, _ip, _ip, _ip, _dp,
                                     _dp]
        L.orc_galerkin_plan.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _ip, C.c_int,
                                        _dp, _ip]
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    """Thread count of the oracle's OpenMP regions (the result does not depend
    on it: the scatter loops are owner-partitioned, see orc.c own_rows)."""
    lib().orc_set_threads(int(n))


def _d(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c_of(a):
    a1, a2, a3 = a
    return np.array([1 / a1 ** 2, 1 / a2 ** 2, 1 / a3 ** 2])


# ----------------------------------------------------------------- element
def shape_grad(xi):
    G = np.zeros((8, 3))
    lib().orc_shape_grad(_d(_f64(xi)), _d(G))
    return G


def element_stiffness(xe, c):
    Ke = np.zeros((8, 8))
    rc = lib().orc_element_stiffness(_d(_f64(xe)), _d(_f64(c)), _d(Ke))
    if rc < 0:
        raise ValueError(f"non-positive Jacobian at Gauss point {-rc - 1}")
    return Ke


def element_stiffness_onepoint(xe, c):
    Ke = np.zeros((8, 8))
    lib().orc_element_stiffness_onepoint(_d(_f64(xe)), _d(_f64(c)), _d(Ke))
    return Ke


def element_rhs(xe, u0):
    fe = np.zeros(8)
    lib().orc_element_rhs(_d(_f64(xe)), _d(_f64(u0)), _d(fe))
    return fe


def element_grad_centre(xe, lam):
    g = np.zeros(3)
    lib().orc_element_grad_centre(_d(_f64(xe)), _d(_f64(lam)), _d(g))
    return g


# ----------------------------------------------------------------- global
def validate_mesh(X, Y, Z):
    n3, n2, n1 = X.shape
    what = C.c_int(0)
    e = lib().orc_validate_mesh(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3,
                                C.byref(what))
    return (None if e < 0 else int(e)), int(what.value)


def assemble(X, Y, Z, a):
    n3, n2, n1 = X.shape
    K = np.zeros((n3, n2, n1, 27))
    rc = lib().orc_assemble(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3,
                            _d(_c_of(a)), _d(K))
    if rc < 0:
        raise ValueError("non-positive Jacobian")
    return K


def assemble_onepoint(X, Y, Z, a):
    n3, n2, n1 = X.shape
    K = np.zeros((n3, n2, n1, 27))
    lib().orc_assemble_onepoint(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3,
                                _d(_c_of(a)), _d(K))
    return K


def rhs(X, Y, Z, u0):
    n3, n2, n1 = X.shape
    f = np.zeros((n3, n2, n1))
    lib().orc_rhs(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3, _d(_f64(u0)), _d(f))
    return f


def d1(X, Y, Z, v):
    n3, n2, n1 = X.shape
    out = np.zeros((n3, n2, n1))
    lib().orc_d1(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3, _d(_f64(v)), _d(out))
    return out


def recover(X, Y, Z, a, lam, u0):
    n3, n2, n1 = X.shape
    u = np.zeros_like(_f64(u0))
    lib().orc_recover(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3, _d(_c_of(a)),
                      _d(_f64(lam)), _d(_f64(u0)), _d(u))
    return u


def apply(K, x):
    n3, n2, n1, _ = K.shape
    y = np.zeros((n3, n2, n1))
    lib().orc_apply(_d(K), n1, n2, n3, _d(_f64(x)), _d(y))
    return y


def residual(K, x, f):
    n3, n2, n1, _ = K.shape
    r = np.zeros((n3, n2, n1))
    nrm = lib().orc_residual(_d(K), n1, n2, n3, _d(_f64(x)), _d(_f64(f)), _d(r))
    return r, nrm


def build_mesh(zs, x0, y0, dx, dy, zeta, H):
    """Terrain-following mesh (orc_build_mesh, reading C13).
    zs: (n2, n1); returns X, Y, Z of shape (n3, n2, n1); raises on H <= zs."""
    zs = _f64(zs)
    zeta = _f64(zeta)
    n2, n1 = zs.shape
    n3 = zeta.size
    X, Y, Z = (np.zeros((n3, n2, n1)) for _ in range(3))
    rc = lib().orc_build_mesh(_d(zs), n1, n2, float(x0), float(y0), float(dx), float(dy),
                              _d(zeta), n3, float(H), _d(X), _d(Y), _d(Z))
    if rc:
        raise ValueError(f"domain top below the terrain at column {rc - 1}")
    return X, Y, Z


def interp_wind(uc, xc0, yc0, DXc, DYc, hc, X, Y, Z):
    """Coarse wind uc (3, nzc, nyc, nxc) at heights above ground hc to element
    centres of the mesh (orc_interp_wind)."""
    uc = _f64(uc)
    hc = _f64(hc)
    _, nzc, nyc, nxc = uc.shape
    n3, n2, n1 = X.shape
    u0 = np.zeros((3, n3 - 1, n2 - 1, n1 - 1))
    rc = lib().orc_interp_wind(_d(uc), nxc, nyc, nzc, float(xc0), float(yc0), float(DXc),
                               float(DYc), _d(hc), _d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2,
                               n3, _d(u0))
    if rc:
        raise ValueError("coarse grid needs >= 2 points per direction")
    return u0


def line_sweep(K, x, f):
    """One vertical line-relaxation sweep (orc_line_sweep)."""
    x = _f64(x).copy()
    K = _f64(K)
    n3, n2, n1 = x.shape
    lib().orc_line_sweep(_d(K), n1, n2, n3, _d(x), _d(_f64(f)))
    return x


SMOOTHERS = {"gs": 0, "line": 1}


def gs_sweep(K, x, f):
    n3, n2, n1, _ = K.shape
    x = _f64(x).copy()
    lib().orc_gs_sweep(_d(K), n1, n2, n3, _d(x), _d(_f64(f)))
    return x


def planner_inputs(X, Y, Z):
    """(h1, h3) the planner starts from (orc_planner_inputs, reading C2):
    h1 = sqrt(dx dy) at the grid origin, h3 = the layer thicknesses of the
    column of minimum Z(i,j,0), ties -> smallest linear index."""
    n3, n2, n1 = X.shape
    h1 = C.c_double(0)
    h3 = np.zeros(n3 - 1)
    lib().orc_planner_inputs(_d(_f64(X)), _d(_f64(Y)), _d(_f64(Z)), n1, n2, n3, C.byref(h1),
                             _d(h3))
    return h1.value, h3


def plan_level(h1, h3, a, rule="coupling_cur", n1=1001, n2=1001):
    h3 = _f64(h3)
    nz = len(h3)
    hflag = C.c_int(0)
    kept = np.zeros(nz + 2, dtype=np.int32)
    nk = C.c_int(0)
    h1n = C.c_double(0)
    h3n = np.zeros(nz + 1)
    any_ = lib().orc_plan_level(h1, _d(h3), nz, a[0], a[1], a[2], RULES[rule], n1, n2,
                                C.byref(hflag), kept.ctypes.data_as(_ip), C.byref(nk),
                                C.byref(h1n), _d(h3n))
    nk = nk.value
    return dict(horizontal=bool(hflag.value), kept=kept[:nk].tolist(), h1=h1n.value,
                h3=h3n[:nk - 1].copy(), coarsens=bool(any_))


def galerkin(Kf, hflag, kept):
    n3, n2, n1, _ = Kf.shape
    kept = np.ascontiguousarray(kept, dtype=np.int32)
    cd = np.zeros(3, dtype=np.int32)
    lib().orc_galerkin_plan(_d(Kf), n1, n2, n3, int(hflag), kept.ctypes.data_as(_ip),
                            len(kept), None, cd.ctypes.data_as(_ip))
    m1, m2, m3 = (int(v) for v in cd)
    Kc = np.zeros((m3, m2, m1, 27))
    rc = lib().orc_galerkin_plan(_d(Kf), n1, n2, n3, int(hflag), kept.ctypes.data_as(_ip),
                                 len(kept), _d(Kc), cd.ctypes.data_as(_ip))
    if rc < 0:
        raise RuntimeError("Galerkin stencil reach > 1")
    return Kc


# ----------------------------------------------------------------- hierarchy
class MG:
    """Oracle multigrid hierarchy on one mesh."""

    def __init__(self, X, Y, Z, a, rule="coupling_cur", coarsest_max_free=4096, pre=2,
                 post=2, smoother="gs", line_from_level=-1):
        self._keep = [_f64(X), _f64(Y), _f64(Z)]
        n3, n2, n1 = X.shape
        err = C.c_int(0)
        L = lib()
        self.h = L.orc_mg_setup(_d(self._keep[0]), _d(self._keep[1]), _d(self._keep[2]), n1,
                                n2, n3, float(a[0]), float(a[1]), float(a[2]), RULES[rule],
                                int(coarsest_max_free), int(pre), int(post), C.byref(err))
        if not self.h:
            raise RuntimeError(f"orc_mg_setup failed, err={err.value}")
        L.orc_mg_set_smoother(self.h, SMOOTHERS[smoother])
        L.orc_mg_set_level_smoother.argtypes = [C.c_void_p, C.c_int, C.c_int]
        self.nlev = L.orc_mg_nlevels(self.h)
        if line_from_level >= 0:   # per-level smoother
            for l in range(line_from_level, self.nlev):
                self.set_level_smoother(l, "line")
        self.coarse_direct = bool(L.orc_mg_coarse_direct(self.h))
        self.dims = []
        for l in range(self.nlev):
            d = np.zeros(3, dtype=np.int32)
            L.orc_mg_level_dims(self.h, l, d.ctypes.data_as(_ip))
            self.dims.append(tuple(int(v) for v in d))
        self.plans = []
        for l in range(self.nlev - 1):
            hf = C.c_int(0)
            kept = np.zeros(300, dtype=np.int32)
            nk = L.orc_mg_plan(self.h, l, C.byref(hf), kept.ctypes.data_as(_ip))
            self.plans.append(dict(horizontal=bool(hf.value), kept=kept[:nk].tolist()))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_mg_free(self.h)
            except TypeError:   # interpreter shutdown: module globals already gone
                pass
            self.h = None

    def set_level_smoother(self, l, smoother):
        """Per-level smoother override ("gs" | "line" | None = the hierarchy's)."""
        lib().orc_mg_set_level_smoother(self.h, int(l), -1 if smoother is None else SMOOTHERS[smoother])

    def shape(self, l):
        n1, n2, n3 = self.dims[l]
        return (n3, n2, n1)

    def K(self, l):
        n1, n2, n3 = self.dims[l]
        p = lib().orc_mg_K(self.h, l)
        return np.ctypeslib.as_array(p, shape=(n3, n2, n1, 27)).copy()

    def gs(self, l, x, f):
        """One sweep of the hierarchy's smoother (point GS or line relaxation)."""
        x = _f64(x).copy()
        lib().orc_mg_gs(self.h, l, _d(x), _d(_f64(f)))
        return x

    def apply(self, l, x):
        y = np.zeros(self.shape(l))
        lib().orc_mg_apply(self.h, l, _d(_f64(x)), _d(y))
        return y

    def restrict(self, l, r):
        fc = np.zeros(self.shape(l + 1))
        lib().orc_mg_restrict(self.h, l, _d(_f64(r)), _d(fc))
        return fc

    def prolong(self, l, xc, x):
        x = _f64(x).copy()
        lib().orc_mg_prolong(self.h, l, _d(_f64(xc)), _d(x))
        return x

    def coarse_solve(self, f):
        x = np.zeros(self.shape(self.nlev - 1))
        lib().orc_mg_coarse_solve(self.h, _d(_f64(f)), _d(x))
        return x

    def vcycle(self, x, f):
        x = _f64(x).copy()
        lib().orc_mg_vcycle(self.h, _d(x), _d(_f64(f)))
        return x

    def solve(self, f, lam0=None, tol=1e-8, max_cycles=100):
        x = np.zeros(self.shape(0))
        hist = np.zeros(max_cycles + 1)
        cyc = C.c_int(0)
        rate = C.c_double(0)
        l0 = None if lam0 is None else _d(_f64(lam0))
        st = lib().orc_mg_solve(self.h, _d(_f64(f)), l0, float(tol), int(max_cycles), _d(x),
                                _d(hist), C.byref(cyc), C.byref(rate))
        c = cyc.value
        return x, dict(status=int(st), cycles=c, hist=hist[:c + 1].copy(), rate=rate.value)

    def work_ratio(self):
        n0 = np.prod(self.dims[0])
        return sum(np.prod(d) for d in self.dims) / n0


# ----------------------------------------------------------------- dense helpers
def free_mask(shape):
    n3, n2, n1 = shape
    m = np.ones(shape, dtype=bool)
    m[-1] = False
    m[:, 0, :] = False
    m[:, -1, :] = False
    m[:, :, 0] = False
    m[:, :, -1] = False
    return m


def stencil_to_dense(K):
    """Full N x N matrix from 27-point storage (all rows, natural couplings)."""
    n3, n2, n1, _ = K.shape
    N = n1 * n2 * n3
    A = np.zeros((N, N))
    for o in range(27):
        dx, dy, dz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
        for k in range(n3):
            kk = k + dz
            if not 0 <= kk < n3:
                continue
            for j in range(n2):
                jj = j + dy
                if not 0 <= jj < n2:
                    continue
                i = np.arange(n1)
                ii = i + dx
                ok = (ii >= 0) & (ii < n1)
                p = (k * n2 + j) * n1 + i[ok]
                q = (kk * n2 + jj) * n1 + ii[ok]
                A[p, q] = K[k, j, i[ok], o]
    return A

"""Python binding of the B200-native wind-downscaling library (``libwd.so``).

Argument marshalling only: every function forwards to the C ABI declared in
``include/wd.h`` (same names), passing raw pointers of torch tensors (device or
host) and the current CUDA stream.  All arithmetic of the hot path runs in the
sm_100a kernels of ``csrc/``; there is no CPU or PyTorch fallback -- importing
this package fails loudly if the shared library is missing.

Paper: Mandel et al., arXiv 2101.08453 (Eq. (3)-(7), Sec. 3).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwd.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build() "
                      "(the CUDA extension is required; there is no fallback)")

_lib = C.CDLL(LIB_PATH)

WD_OK, WD_E_INVAL, WD_E_MESH, WD_E_NOCONV, WD_E_DIVERGED, WD_E_NONFINITE, WD_E_CUDA, \
    WD_E_NCCL, WD_E_OOM, WD_E_INTERNAL = range(10)
RULES = {"coupling_cur": 0, "coupling_paper": 1, "verbatim": 2, "full": 3}
SMOOTHERS = {"fused": 0, "phased": 1, "line": 2}
ERRNAMES = {1: "WD_E_INVAL", 2: "WD_E_MESH", 3: "WD_E_NOCONV", 4: "WD_E_DIVERGED",
            5: "WD_E_NONFINITE", 6: "WD_E_CUDA", 7: "WD_E_NCCL", 8: "WD_E_OOM",
            9: "WD_E_INTERNAL"}


class wd_options(C.Structure):
    _fields_ = [("pre_smooth", C.c_int), ("post_smooth", C.c_int), ("max_cycles", C.c_int),
                ("coarsest_max_free", C.c_int), ("coarse_iters", C.c_int),
                ("coarsen_rule", C.c_int), ("use_graph", C.c_int),
                ("gather_below_nodes", C.c_longlong), ("rank", C.c_int), ("nranks", C.c_int),
                ("nccl_comm", C.c_void_p), ("j_begin", C.c_int), ("j_end", C.c_int),
                ("profile", C.c_int), ("smoother", C.c_int), ("line_from_level", C.c_int),
                ("device_loop", C.c_int), ("overlap_halo", C.c_int)]


class wd_report(C.Structure):
    _fields_ = [("status", C.c_int), ("cycles", C.c_int), ("converged", C.c_int),
                ("nlevels", C.c_int), ("rel_res0", C.c_double), ("rel_res_final", C.c_double),
                ("rate", C.c_double), ("rel_res_hist", C.c_double * 256),
                ("dims", (C.c_int * 3) * 32), ("coarse_direct", C.c_int),
                ("coarse_free", C.c_int)]

    def to_dict(self):
        c = self.cycles
        return dict(status=self.status, cycles=c, converged=bool(self.converged),
                    nlevels=self.nlevels, rel_res0=self.rel_res0,
                    rel_res_final=self.rel_res_final, rate=self.rate,
                    hist=[self.rel_res_hist[t] for t in range(min(c, 255) + 1)],
                    dims=[tuple(self.dims[l]) for l in range(self.nlevels)],
                    coarse_direct=bool(self.coarse_direct), coarse_free=self.coarse_free)


_vp = C.c_void_p
_dp = C.c_void_p
_lib.wd_default_options.argtypes = [C.POINTER(wd_options)]
_lib.wd_last_error.restype = C.c_char_p
_lib.wd_assemble.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                             C.c_double, C.POINTER(wd_options), _vp, C.POINTER(_vp)]
_lib.wd_rhs.argtypes = [_vp, _dp, _dp, _vp]
_lib.wd_vcycle.argtypes = [_vp, _dp, _dp, C.POINTER(C.c_double), _vp]
_lib.wd_solve.argtypes = [_vp, _dp, _dp, C.c_double, _dp, C.POINTER(wd_report), _vp]
_lib.wd_recover_wind.argtypes = [_vp, _dp, _dp, _dp, _vp]
_lib.wd_destroy.argtypes = [_vp]
_lib.wd_device_bytes.argtypes = [_vp]
_lib.wd_device_bytes.restype = C.c_longlong
_lib.wd_num_levels.argtypes = [_vp]
_lib.wd_level_dims.argtypes = [_vp, C.c_int, C.POINTER(C.c_int)]
_lib.wd_level_plan.argtypes = [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int)]
_lib.wd_get_stencil.argtypes = [_vp, C.c_int, _dp, _vp]
_lib.wd_apply.argtypes = [_vp, C.c_int, _dp, _dp, _vp]
_lib.wd_smooth.argtypes = [_vp, C.c_int, _dp, _dp, C.c_int, _vp]
_lib.wd_restrict.argtypes = [_vp, C.c_int, _dp, _dp, _vp]
_lib.wd_prolong.argtypes = [_vp, C.c_int, _dp, _dp, _vp]
_lib.wd_coarse_solve.argtypes = [_vp, _dp, _dp, _vp]
_lib.wd_residual_norm.argtypes = [_vp, _dp, _dp, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), _vp]

_lib.wd_profile_read.argtypes = [_vp, C.POINTER(C.c_double), C.c_int]
_lib.wd_profile_reset.argtypes = [_vp]
_lib.wd_launch_count.restype = C.c_longlong
_lib.wd_bench_kernel.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
_lib.wd_partition_rows.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
_lib.wd_nccl_unique_id.argtypes = [C.c_char_p]
_lib.wd_nccl_comm_init.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
_lib.wd_gather_level.argtypes = [_vp]
_lib.wd_build_mesh.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                               C.c_double, _dp, C.c_int, C.c_double, _dp, _dp, _dp, _vp]
_lib.wd_interp_wind.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_double, _dp, _dp, _dp, _dp, C.c_int, C.c_int,
                                C.c_int, _dp, _vp]
_lib.wd_mass_consistency.argtypes = [_vp, _dp, C.POINTER(C.c_double), _vp]
_lib.wd_downscale_step.argtypes = [_vp, _dp, _dp, C.c_int, C.c_double, _dp, C.POINTER(wd_report),
                                   _vp]

# every symbol include/wd.h declares
ABI_SYMBOLS = ["wd_default_options", "wd_assemble", "wd_rhs", "wd_vcycle", "wd_solve",
               "wd_recover_wind", "wd_destroy", "wd_last_error", "wd_device_bytes",
               "wd_num_levels", "wd_level_dims", "wd_level_plan", "wd_get_stencil",
               "wd_apply", "wd_smooth", "wd_restrict", "wd_prolong", "wd_coarse_solve",
               "wd_residual_norm", "wd_profile_read", "wd_profile_reset", "wd_launch_count",
               "wd_bench_kernel", "wd_partition_rows", "wd_nccl_unique_id", "wd_nccl_comm_init",
               "wd_gather_level", "wd_build_mesh", "wd_interp_wind", "wd_mass_consistency",
               "wd_downscale_step", "wd_plan_decomposition"]

BENCH_KERNELS = {"gs_sweep": 0, "apply": 1, "restrict": 2, "prolong": 3, "vcycle": 4,
                 "residual_norm": 5, "galerkin": 6, "assemble": 7, "gs_sweep_phased": 8,
                 "gs_sweep_res": 9}


class WDError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRNAMES.get(code, code)}: {msg}")
        self.code = code


def last_error() -> str:
    return _lib.wd_last_error().decode()


def _check(rc, ok=(WD_OK,)):
    if rc not in ok:
        raise WDError(rc, last_error())
    return rc


def _ptr(t: torch.Tensor):
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_contiguous():
        raise WDError(WD_E_INVAL, "arguments must be contiguous float64 tensors "
                      f"(got {getattr(t, 'dtype', type(t))})")
    return C.c_void_p(t.data_ptr())


def _arg(ctx: "Context", t: torch.Tensor, shape, name: str):
    """Validate a tensor crossing the ABI against the context: the C side takes
    every size from the context, so a wrong shape or another GPU's tensor would
    read or write out of bounds.  Host tensors are allowed (staged inside)."""
    if not isinstance(t, torch.Tensor):
        raise WDError(WD_E_INVAL, f"{name}: expected a torch.Tensor")
    if tuple(t.shape) != tuple(shape):
        raise WDError(WD_E_INVAL, f"{name}: shape {tuple(t.shape)} != expected {tuple(shape)}")
    if t.is_cuda and t.device != ctx.device:
        raise WDError(WD_E_INVAL, f"{name}: on {t.device}, context on {ctx.device}")
    return _ptr(t)


def _stream(t: torch.Tensor):
    if t.is_cuda:
        return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)
    return C.c_void_p(0)


def default_options(**kw) -> wd_options:
    o = wd_options()
    _lib.wd_default_options(C.byref(o))
    for k, v in kw.items():
        if k == "coarsen_rule" and isinstance(v, str):
            v = RULES[v]
        if k == "smoother" and isinstance(v, str):
            v = SMOOTHERS[v]
        setattr(o, k, v)
    return o


class Context:
    """Owns a ``wd_ctx*`` (hierarchy and workspaces on the device)."""

    def __init__(self, handle, dims, device, rows=None):
        self.h = handle
        self.dims = dims        # global node dims (n1, n2, n3)
        self.device = device
        self.rows = rows if rows is not None else dims[1]   # node rows of the ABI arrays
        self._destroy = _lib.wd_destroy   # module globals may be gone at interpreter exit

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    @property
    def node_shape(self):
        """Shape of the node arrays of the ABI calls (a slab in NCCL mode)."""
        n1, _, n3 = self.dims
        return (n3, self.rows, n1)

    @property
    def elem_shape(self):
        n1, _, n3 = self.dims
        return (3, n3 - 1, self.rows - 1, n1 - 1)

    def device_bytes(self):
        return int(_lib.wd_device_bytes(self.h))

    def num_levels(self):
        return int(_lib.wd_num_levels(self.h))

    def level_dims(self, l):
        d = (C.c_int * 3)()
        _check(_lib.wd_level_dims(self.h, l, d))
        return tuple(d)

    def level_shape(self, l):
        n1, n2, n3 = self.level_dims(l)
        return (n3, n2, n1)

    def level_plan(self, l):
        hz = C.c_int()
        kept = (C.c_int * 600)()
        nk = C.c_int()
        _check(_lib.wd_level_plan(self.h, l, C.byref(hz), kept, C.byref(nk)))
        return dict(horizontal=bool(hz.value), kept=list(kept[:nk.value]))


def wd_profile_read(ctx: Context):
    out = (C.c_double * 12)()
    _lib.wd_profile_read(ctx.h, out, 12)
    keys = ("gs0_ms", "gs0_sweeps", "vcycle_ms", "vcycles", "resid_ms", "resids", "gs0res_ms",
            "gs0res_sweeps", "apply0_ms", "apply0_launches", "gs0_sweeps_all",
            "gs0res_sweeps_all")
    return dict(zip(keys, list(out)))


def wd_profile_reset(ctx: Context):
    _lib.wd_profile_reset(ctx.h)


def wd_launch_count() -> int:
    return int(_lib.wd_launch_count())


def wd_bench_kernel(ctx: Context, which, level=0, reps=10) -> float:
    ms = C.c_double()
    w = BENCH_KERNELS[which] if isinstance(which, str) else int(which)
    _check(_lib.wd_bench_kernel(ctx.h, w, level, reps, C.byref(ms)))
    return ms.value


def wd_partition_rows(n2, nranks, rank):
    """Owned node rows [j_begin, j_end) of `rank` (even split, wd.h)."""
    a, b = C.c_int(), C.c_int()
    _lib.wd_partition_rows(int(n2), int(nranks), int(rank), C.byref(a), C.byref(b))
    return a.value, b.value


def slab_rows(n2, nranks, rank, halo=2):
    """Rows [lo, hi) of the arrays a rank passes in NCCL mode (owned + halo)."""
    a, b = wd_partition_rows(n2, nranks, rank)
    return max(a - halo, 0), min(b + halo, n2)


_lib.wd_plan_decomposition.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.POINTER(C.c_double),
                                       C.POINTER(wd_options), C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.c_int,
                                       C.POINTER(C.c_int)]


def wd_plan_decomposition(dims, a, h1, h3, nranks, rank, w=1, opt: wd_options | None = None):
    """Host-only slab-decomposition plan (wd.h wd_plan_decomposition): the
    hierarchy and this rank's rows per level, the gather level and the halo
    messages of one w-row exchange.  No GPU needed."""
    n1, n2, n3 = dims
    h3a = (C.c_double * (n3 - 1))(*[float(v) for v in h3])
    o = opt if opt is not None else default_options()
    nl, ga, nm = C.c_int(), C.c_int(), C.c_int()
    lev = (C.c_int * (8 * 32))()
    msgs = (C.c_int * (5 * 4 * 32))()
    _check(_lib.wd_plan_decomposition(int(n1), int(n2), int(n3), float(a[0]), float(a[1]),
                                      float(a[2]), float(h1), h3a, C.byref(o), int(nranks),
                                      int(rank), int(w), C.byref(nl), C.byref(ga), lev, 32, msgs,
                                      4 * 32, C.byref(nm)))
    levels = []
    for l in range(nl.value):
        v = lev[8 * l: 8 * l + 8]
        levels.append(dict(dims=tuple(v[0:3]), dist=bool(v[3]), held=(v[4], v[5]),
                           owned=(v[6], v[7])))
    ms = [dict(level=msgs[5 * m], peer=msgs[5 * m + 1], send=bool(msgs[5 * m + 2]),
               row0=msgs[5 * m + 3], rows=msgs[5 * m + 4]) for m in range(nm.value)]
    return dict(nlevels=nl.value, gather=ga.value, levels=levels, msgs=ms)


def wd_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.wd_nccl_unique_id(buf))
    return buf.raw


def wd_nccl_comm_init(uid: bytes, nranks, rank):
    comm = C.c_void_p()
    _check(_lib.wd_nccl_comm_init(C.c_char_p(uid), int(nranks), int(rank), C.byref(comm)))
    return comm


def nccl_comm_from_torch(group=None):
    """One communicator per process group: rank 0 draws the unique id, the
    torch process group broadcasts it (plumbing only)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [wd_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return wd_nccl_comm_init(obj[0], world, rank)


def wd_gather_level(ctx: "Context") -> int:
    return int(_lib.wd_gather_level(ctx.h))


# ------------------------------------------------------------------ ABI calls
def wd_assemble(X, Y, Z, a, opt: wd_options | None = None, n2_global=None) -> Context:
    """X, Y, Z: node arrays (n3, rows, n1); rows = n2 except in NCCL mode, where
    they hold this rank's slab (slab_rows) and n2_global gives the grid's n2."""
    n3, rows, n1 = X.shape
    for name, t in (("Y", Y), ("Z", Z)):
        if tuple(t.shape) != tuple(X.shape) or t.device != X.device:
            raise WDError(WD_E_INVAL, f"{name}: shape/device differ from X")
    n2 = int(n2_global) if n2_global is not None else rows
    h = C.c_void_p()
    o = opt if opt is not None else default_options()
    _check(_lib.wd_assemble(_ptr(X), _ptr(Y), _ptr(Z), n1, n2, n3, float(a[0]), float(a[1]),
                            float(a[2]), C.byref(o), _stream(X), C.byref(h)))
    return Context(h, (n1, n2, n3), X.device, rows)


def wd_rhs(ctx: Context, u0, f=None):
    if f is None:
        f = torch.empty(ctx.node_shape, dtype=torch.float64, device=u0.device)
    _check(_lib.wd_rhs(ctx.h, _arg(ctx, u0, ctx.elem_shape, "u0"),
                       _arg(ctx, f, ctx.node_shape, "f"), _stream(u0)))
    return f


def wd_vcycle(ctx: Context, lam, f, want_residual=True):
    rel = C.c_double(0)
    _check(_lib.wd_vcycle(ctx.h, _arg(ctx, lam, ctx.node_shape, "lam"),
                          _arg(ctx, f, ctx.node_shape, "f"),
                          C.byref(rel) if want_residual else None, _stream(lam)))
    return rel.value if want_residual else None


def wd_solve(ctx: Context, f, lam0=None, rel_tol=1e-8, lam=None, raise_on_noconv=True):
    if lam is None:
        lam = torch.empty(ctx.node_shape, dtype=torch.float64, device=f.device)
    rep = wd_report()
    rc = _lib.wd_solve(ctx.h, _arg(ctx, f, ctx.node_shape, "f"),
                       None if lam0 is None else _arg(ctx, lam0, ctx.node_shape, "lam0"),
                       float(rel_tol), _arg(ctx, lam, ctx.node_shape, "lam"), C.byref(rep),
                       _stream(f))
    ok = (WD_OK,) if raise_on_noconv else (WD_OK, WD_E_NOCONV, WD_E_DIVERGED, WD_E_NONFINITE)
    _check(rc, ok)
    return lam, rep.to_dict()


def wd_recover_wind(ctx: Context, lam, u0, u=None):
    if u is None:
        u = torch.empty_like(u0)
    _check(_lib.wd_recover_wind(ctx.h, _arg(ctx, lam, ctx.node_shape, "lam"),
                                _arg(ctx, u0, ctx.elem_shape, "u0"),
                                _arg(ctx, u, ctx.elem_shape, "u"), _stream(u0)))
    return u


# ------------------------------------------------------------------ inspection
def wd_get_stencil(ctx: Context, level=0, device=None):
    n3, n2, n1 = ctx.level_shape(level)
    K = torch.empty((n3, n2, n1, 27), dtype=torch.float64, device=device or ctx.device)
    _check(_lib.wd_get_stencil(ctx.h, level, _arg(ctx, K, (n3, n2, n1, 27), "K"), _stream(K)))
    return K


def wd_apply(ctx: Context, level, x, y=None):
    y = torch.empty_like(x) if y is None else y
    sh = ctx.level_shape(level)
    _check(_lib.wd_apply(ctx.h, level, _arg(ctx, x, sh, "x"), _arg(ctx, y, sh, "y"), _stream(x)))
    return y


def wd_smooth(ctx: Context, level, x, f, sweeps=1):
    sh = ctx.level_shape(level)
    _check(_lib.wd_smooth(ctx.h, level, _arg(ctx, x, sh, "x"), _arg(ctx, f, sh, "f"),
                          int(sweeps), _stream(x)))
    return x


def wd_restrict(ctx: Context, level, r, fc=None):
    if fc is None:
        fc = torch.empty(ctx.level_shape(level + 1), dtype=torch.float64, device=r.device)
    _check(_lib.wd_restrict(ctx.h, level, _arg(ctx, r, ctx.level_shape(level), "r"),
                            _arg(ctx, fc, ctx.level_shape(level + 1), "fc"), _stream(r)))
    return fc


def wd_prolong(ctx: Context, level, xc, x):
    _check(_lib.wd_prolong(ctx.h, level, _arg(ctx, xc, ctx.level_shape(level + 1), "xc"),
                           _arg(ctx, x, ctx.level_shape(level), "x"), _stream(x)))
    return x


def wd_coarse_solve(ctx: Context, f, x=None):
    x = torch.empty_like(f) if x is None else x
    sh = ctx.level_shape(ctx.num_levels() - 1)
    _check(_lib.wd_coarse_solve(ctx.h, _arg(ctx, f, sh, "f"), _arg(ctx, x, sh, "x"), _stream(f)))
    return x


def wd_residual_norm(ctx: Context, x, f):
    a = C.c_double()
    r = C.c_double()
    _check(_lib.wd_residual_norm(ctx.h, _arg(ctx, x, ctx.node_shape, "x"),
                                 _arg(ctx, f, ctx.node_shape, "f"), C.byref(a), C.byref(r),
                                 _stream(x)))
    return a.value, r.value


def downscale(X, Y, Z, u0, a, rel_tol=1e-8, lam0=None, opt=None):
    """End to end through the public ABI: assemble, RHS, solve, recover.
    Inputs may be host or device tensors (host buffers are staged inside the
    library calls).  Returns (u, lam, report)."""
    ctx = wd_assemble(X, Y, Z, a, opt)
    try:
        f = wd_rhs(ctx, u0, torch.empty(ctx.node_shape, dtype=torch.float64, device=u0.device))
        lam, rep = wd_solve(ctx, f, lam0, rel_tol)
        u = wd_recover_wind(ctx, lam, u0)
    finally:
        ctx.close()
    return u, lam, rep


# ------------------------------------------------------------------ f4: either side of the path
def _host_f64(a):
    import numpy as np
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def wd_build_mesh(zs: torch.Tensor, x0, y0, dx, dy, zeta, H):
    """Terrain-following mesh (wd.h wd_build_mesh): zs (n2, n1) tensor on the
    device or host; zeta: the n3 level heights (host sequence); returns X, Y, Z
    of shape (n3, n2, n1) on zs's device."""
    z = _host_f64(zeta)
    n2, n1 = zs.shape
    n3 = z.size
    X, Y, Z = (torch.empty((n3, n2, n1), dtype=torch.float64, device=zs.device) for _ in range(3))
    _check(_lib.wd_build_mesh(_ptr(zs), n1, n2, float(x0), float(y0), float(dx), float(dy),
                              z.ctypes.data_as(C.c_void_p), n3, float(H), _ptr(X), _ptr(Y),
                              _ptr(Z), _stream(zs)))
    return X, Y, Z


def wd_interp_wind(uc: torch.Tensor, xc0, yc0, DXc, DYc, hc, X, Y, Z):
    """Coarse wind uc (3, nzc, nyc, nxc) at heights above ground hc (host
    sequence) to the element centres of the mesh X, Y, Z (wd_interp_wind)."""
    h = _host_f64(hc)
    _, nzc, nyc, nxc = uc.shape
    n3, n2, n1 = X.shape
    for name, t in (("Y", Y), ("Z", Z)):
        if tuple(t.shape) != tuple(X.shape) or t.device != X.device:
            raise WDError(WD_E_INVAL, f"{name}: shape/device differ from X")
    u0 = torch.empty((3, n3 - 1, n2 - 1, n1 - 1), dtype=torch.float64, device=X.device)
    _check(_lib.wd_interp_wind(_ptr(uc), nxc, nyc, nzc, float(xc0), float(yc0), float(DXc),
                               float(DYc), h.ctypes.data_as(C.c_void_p), _ptr(X), _ptr(Y), _ptr(Z),
                               n1, n2, n3, _ptr(u0), _stream(X)))
    return u0


def wd_mass_consistency(ctx: Context, u):
    """(l2, max) of the one-point weak divergence D1(u) over free nodes."""
    out = (C.c_double * 2)()
    _check(_lib.wd_mass_consistency(ctx.h, _arg(ctx, u, ctx.elem_shape, "u"), out, _stream(u)))
    return float(out[0]), float(out[1])


def wd_downscale_step(ctx: Context, u0, lam, warm=True, rel_tol=1e-8, u=None,
                      raise_on_noconv=True):
    """RHS + (warm-started) solve + wind recovery in one call; lam is updated
    in place.  Returns (u, report)."""
    if u is None:
        u = torch.empty_like(u0)
    rep = wd_report()
    rc = _lib.wd_downscale_step(ctx.h, _arg(ctx, u0, ctx.elem_shape, "u0"),
                                _arg(ctx, lam, ctx.node_shape, "lam"), 1 if warm else 0,
                                float(rel_tol), _arg(ctx, u, ctx.elem_shape, "u"), C.byref(rep),
                                _stream(u0))
    ok = (WD_OK,) if raise_on_noconv else (WD_OK, WD_E_NOCONV, WD_E_DIVERGED, WD_E_NONFINITE)
    _check(rc, ok)
    return u, rep.to_dict()

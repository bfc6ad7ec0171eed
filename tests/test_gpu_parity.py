"""GPU (sm_100a) vs oracle parity through the C ABI, element by element on the
same seeded inputs.  Tolerances (BASELINE.json north_star, normalisations of
DESIGN.md "Parity tolerances"):
  * operator apply, RHS, recovery, stencil entries: <= 1e-12 relative max;
  * one GS sweep, restriction, prolongation: <= 1e-11 relative max;
  * one V-cycle: <= 1e-10 relative max (SURVEY 8(c) asked 1e-12; the coarsest
    direct solves differ -- dense Cholesky in the oracle, an explicit
    Gauss-Jordan inverse on the GPU, reading C8 -- and agree only to
    O(cond(K_c) eps), which the prolongation carries into the fine iterate);
  * lambda after both solves reach rel. residual 1e-10: <= 1e-8 relative l2;
  * V-cycle convergence factor within 10 %.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from brute import free_mask, free_pair_mask, stencil_asymmetry

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def _n(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_max(a, b, scale=None):
    s = np.abs(b).max() if scale is None else scale
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


CASES = {
    "tiny": lambda: synth.tiny(),
    "tiny_a3": lambda: (lambda p: synth.Problem(p.name, p.nx, p.ny, p.nz, p.X, p.Y, p.Z, p.u0,
                                                (1.0, 2.0, 7.0), p.meta))(synth.tiny()),
    "small": lambda: synth.small(),
    "ragged": lambda: synth.hill(nx=37, ny=22, nz=5, dx=40.0, height=120.0, sigma=300.0,
                                 dz0=8.0, r=1.3, a=(1, 1, 3)),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request, wd):
    p = CASES[request.param]()
    X, Y, Z, u0 = p.numpy()
    cmax = 60 if p.name != "small" else 4096
    opt = wd.default_options(coarsest_max_free=cmax)
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=cmax)
    yield dict(p=p, np=(X, Y, Z, u0), g=g, ctx=ctx, mg=mg)
    ctx.close()


def test_hierarchy_matches(case):
    ctx, mg = case["ctx"], case["mg"]
    assert ctx.num_levels() == mg.nlev
    for l in range(mg.nlev):
        assert ctx.level_dims(l) == mg.dims[l]
    for l in range(mg.nlev - 1):
        assert ctx.level_plan(l) == mg.plans[l]


def test_stencil_parity_all_levels(case, wd):
    ctx, mg = case["ctx"], case["mg"]
    for l in range(mg.nlev):
        Kg = _n(wd.wd_get_stencil(ctx, l))
        Ko = mg.K(l)
        if l == 0:
            err = rel_max(Kg, Ko)                 # every row, natural couplings
        else:                                     # Galerkin: free rows, free columns
            m = free_pair_mask(mg.shape(l))
            err = rel_max(Kg[m], Ko[m])
        assert err <= 1e-12, (l, err)
        # exact symmetry of the stored operator (each pair stored once)
        assert stencil_asymmetry(Kg) == 0.0, l


def test_rhs_parity(case, wd):
    X, Y, Z, u0 = case["np"]
    f = _n(wd.wd_rhs(case["ctx"], case["g"].u0))
    fo = oracle.rhs(X, Y, Z, u0)
    assert rel_max(f, fo) <= 1e-12


def test_apply_parity_all_levels(case, wd):
    """C16: lambda ~ U[-1,1] on free nodes, error / max|K lambda|."""
    ctx, mg = case["ctx"], case["mg"]
    for l in range(mg.nlev):
        x = np.random.default_rng(l).uniform(-1, 1, mg.shape(l)) * free_mask(mg.shape(l))
        y = _n(wd.wd_apply(ctx, l, _t(x)))
        yo = mg.apply(l, x)
        assert rel_max(y, yo) <= 1e-12, l


def test_recover_parity(case, wd):
    X, Y, Z, u0 = case["np"]
    p = case["p"]
    lam = synth.random_lambda(p, 5).numpy() * 100.0
    u = _n(wd.wd_recover_wind(case["ctx"], _t(lam), case["g"].u0))
    uo = oracle.recover(X, Y, Z, p.a, lam, u0)
    assert rel_max(u, uo) <= 1e-12


def test_smoother_transfer_parity(case, wd):
    ctx, mg = case["ctx"], case["mg"]
    rng = np.random.default_rng(7)
    for l in range(mg.nlev):
        s = mg.shape(l)
        fm = free_mask(s)
        x = rng.uniform(-1, 1, s) * fm
        f = rng.uniform(-1, 1, s) * fm
        xg = _n(wd.wd_smooth(ctx, l, _t(x), _t(f), sweeps=1))
        xo = mg.gs(l, x, f)
        assert rel_max(xg, xo) <= 1e-11, ("gs", l)
        if l < mg.nlev - 1:
            fc = _n(wd.wd_restrict(ctx, l, _t(x)))
            assert rel_max(fc, mg.restrict(l, x)) <= 1e-13, ("restrict", l)
            sc = mg.shape(l + 1)
            xc = rng.uniform(-1, 1, sc) * free_mask(sc)
            xp = _n(wd.wd_prolong(ctx, l, _t(xc), _t(x)))
            assert rel_max(xp, mg.prolong(l, xc, x)) <= 1e-14, ("prolong", l)


def test_coarse_solve_parity(case, wd):
    ctx, mg = case["ctx"], case["mg"]
    s = mg.shape(mg.nlev - 1)
    f = np.random.default_rng(3).normal(size=s) * free_mask(s)
    x = _n(wd.wd_coarse_solve(ctx, _t(f)))
    assert rel_max(x, mg.coarse_solve(f)) <= 1e-10


def test_vcycle_parity(case, wd):
    ctx, mg = case["ctx"], case["mg"]
    X, Y, Z, u0 = case["np"]
    f = oracle.rhs(X, Y, Z, u0)
    lam0 = synth.random_lambda(case["p"], 11).numpy()
    lam = _t(lam0)
    for c in range(3):
        wd.wd_vcycle(ctx, lam, _t(f))
        lam0 = mg.vcycle(lam0, f)
        # 1e-10, not 1e-12: Cholesky (oracle) vs Gauss-Jordan inverse (GPU) at
        # the coarsest level agree to O(cond(K_c) eps) only (reading C8)
        assert rel_max(_n(lam), lam0) <= 1e-10, c


def test_solve_parity(case, wd):
    """lambda after both solves reach 1e-10: <= 1e-8 rel l2; rate within 10 %;
    recovered wind <= 1e-8 rel l2."""
    ctx, mg, p = case["ctx"], case["mg"], case["p"]
    X, Y, Z, u0 = case["np"]
    f = wd.wd_rhs(ctx, case["g"].u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
    fo = oracle.rhs(X, Y, Z, u0)
    lo, ro = mg.solve(fo, tol=1e-10, max_cycles=100)
    assert rep["converged"] and ro["status"] == 0
    ln = _n(lam)
    assert np.linalg.norm(ln - lo) / np.linalg.norm(lo) <= 1e-8
    if ro["cycles"] >= 3:
        assert abs(rep["rate"] - ro["rate"]) <= 0.1 * ro["rate"]
    assert abs(rep["cycles"] - ro["cycles"]) <= 1
    u = _n(wd.wd_recover_wind(ctx, lam, case["g"].u0))
    uo = oracle.recover(X, Y, Z, p.a, lo, u0)
    assert np.linalg.norm(u - uo) / np.linalg.norm(uo) <= 1e-8
    # warm start from the converged lambda: <= 1 cycle
    _, rep2 = wd.wd_solve(ctx, f, lam0=lam, rel_tol=1e-10)
    assert rep2["cycles"] <= 1
    # deterministic: bitwise-equal re-solve
    lam3, _ = wd.wd_solve(ctx, f, rel_tol=1e-10)
    assert torch.equal(lam3, lam)


def test_divergence_identity_gpu_wind(case, wd):
    """C12: D1(u_gpu) - (K1 - K) lambda = K lambda - f at free nodes, with the
    wind recovered on the GPU and D1, K1, K from the oracle."""
    ctx, p = case["ctx"], case["p"]
    X, Y, Z, u0 = case["np"]
    f = wd.wd_rhs(ctx, case["g"].u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-9)
    u = _n(wd.wd_recover_wind(ctx, lam, case["g"].u0))
    ln = _n(lam)
    K = oracle.assemble(X, Y, Z, p.a)
    K1 = oracle.assemble_onepoint(X, Y, Z, p.a)
    fo = oracle.rhs(X, Y, Z, u0)
    lhs = oracle.d1(X, Y, Z, u) - (oracle.apply(K1, ln) - oracle.apply(K, ln))
    r = oracle.apply(K, ln) - fo
    fm = free_mask(X.shape)
    assert np.abs(lhs - r)[fm].max() <= 1e-10 * np.abs(fo).max()
    assert np.linalg.norm(r[fm]) / np.linalg.norm(fo) <= 1.01e-9


def test_host_pointer_path(wd):
    """The same ABI calls with host (CPU) tensors stage through the device and
    give bitwise the same results."""
    p = synth.tiny()
    g = p.to(DEV)
    opt = wd.default_options(coarsest_max_free=60)
    ctx_d = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    ctx_h = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)
    fd = wd.wd_rhs(ctx_d, g.u0)
    fh = wd.wd_rhs(ctx_h, p.u0)
    assert torch.equal(fd.cpu(), fh)
    ld, _ = wd.wd_solve(ctx_d, fd, rel_tol=1e-9)
    lh, _ = wd.wd_solve(ctx_h, fh, rel_tol=1e-9)
    assert torch.equal(ld.cpu(), lh)
    ud = wd.wd_recover_wind(ctx_d, ld, g.u0)
    uh = wd.wd_recover_wind(ctx_h, lh, p.u0)
    assert torch.equal(ud.cpu(), uh)


def test_mesh_error_reported(wd):
    p = synth.tiny()
    Z = p.Z.clone()
    Z[3, 5, 7], Z[4, 5, 7] = p.Z[4, 5, 7].item(), p.Z[3, 5, 7].item()
    g = p.to(DEV)
    with pytest.raises(wd.WDError) as e:
        wd.wd_assemble(g.X, g.Y, Z.to(DEV), p.a)
    assert e.value.code == wd.WD_E_MESH
    assert "(6,4,3)" in wd.last_error()


def test_zero_rhs_and_noconv(wd):
    p = synth.tiny()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=60,
                                                                 max_cycles=2))
    f = torch.zeros(ctx.node_shape, dtype=torch.float64, device=DEV)
    lam, rep = wd.wd_solve(ctx, f, lam0=torch.ones_like(f))
    assert rep["cycles"] == 0 and not lam.any()
    f = wd.wd_rhs(ctx, g.u0)
    with pytest.raises(wd.WDError) as e:
        wd.wd_solve(ctx, f, rel_tol=1e-14)
    assert e.value.code == wd.WD_E_NOCONV
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-14, raise_on_noconv=False)
    assert rep["cycles"] == 2 and not rep["converged"]


@pytest.mark.parametrize("rule", ["coupling_cur", "coupling_paper", "verbatim", "full"])
def test_rules_hierarchy_and_solve(wd, rule):
    p = synth.hill(nx=32, ny=32, nz=8, a=(1, 1, 10))
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=100,
                                                                 coarsen_rule=rule))
    mg = oracle.MG(X, Y, Z, p.a, rule=rule, coarsest_max_free=100)
    assert [ctx.level_dims(l) for l in range(ctx.num_levels())] == mg.dims
    f = wd.wd_rhs(ctx, g.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10, raise_on_noconv=False)
    lo, ro = mg.solve(oracle.rhs(X, Y, Z, u0), tol=1e-10, max_cycles=100)
    assert rep["cycles"] == ro["cycles"]
    if ro["status"] == 0:
        assert np.linalg.norm(_n(lam) - lo) / np.linalg.norm(lo) <= 1e-8


def test_warm_start_sequence_parity(case, wd):
    """BASELINE configs[4] in miniature: u0 perturbed by a smooth
    increment, each solve warm-started from the previous lambda, on both
    sides: lambda <= 1e-8 rel l2 and the same number of cycles (+-1) at every
    step, initial residuals within 1e-10 relative."""
    ctx, mg, p = case["ctx"], case["mg"], case["p"]
    X, Y, Z, u0 = case["np"]
    rng = np.random.default_rng(31)
    nz, ny, nx = u0.shape[1:]
    yy, xx = np.meshgrid(np.linspace(0, 1, ny), np.linspace(0, 1, nx), indexing="ij")
    lam_g, lam_o = None, None
    u = u0.copy()
    for step in range(3):
        a, b = rng.normal(0, 0.5, 2)
        u[0] += a * np.sin(np.pi * xx)[None] * np.cos(np.pi * yy)[None]
        u[1] += b * np.cos(np.pi * xx)[None] * np.sin(np.pi * yy)[None]
        fo = oracle.rhs(X, Y, Z, u)
        lo, ro = mg.solve(fo, lam0=lam_o, tol=1e-10, max_cycles=100)
        fg = wd.wd_rhs(ctx, _t(u))
        lg, rg = wd.wd_solve(ctx, fg, lam0=lam_g, rel_tol=1e-10)
        ln = _n(lg)
        assert np.linalg.norm(ln - lo) <= 1e-8 * np.linalg.norm(lo), step
        assert abs(rg["cycles"] - ro["cycles"]) <= 1, (step, rg["cycles"], ro["cycles"])
        assert abs(rg["rel_res0"] - ro["hist"][0]) <= 1e-10 * max(ro["hist"][0], 1e-300), step
        lam_g, lam_o = lg, lo

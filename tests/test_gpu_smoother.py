"""The fused one-pass sweep (k_gs_fused.cu) against the four colour-phase
launches (k_mg.cu) and the oracle.

The two GPU schedules perform the same floating-point operations in the same
order for every node (P:174-176 smoother, colour order of reading C7), so the
iterates must agree BIT FOR BIT on every level, for any number of sweeps and
any tile raggedness; the oracle agreement (<= 1e-11 relative max per sweep) is
in test_gpu_parity.py, which runs the default (fused) smoother.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from brute import free_mask

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


GRIDS = {
    "tiny": lambda: synth.tiny(),
    "small": lambda: synth.small(),
    # ragged in i and j against the 64 x 8 tile, odd and even node counts
    "ragged_a": lambda: synth.hill(nx=150, ny=77, nz=9, dx=40.0, height=200.0, sigma=600.0,
                                   dz0=8.0, r=1.2, a=(1, 1, 10)),
    "ragged_b": lambda: synth.hill(nx=65, ny=9, nz=3, dx=30.0, height=80.0, sigma=200.0,
                                   dz0=5.0, r=1.1, a=(1, 2, 3)),
    "thin": lambda: synth.hill(nx=3, ny=40, nz=15, dx=30.0, height=50.0, sigma=100.0,
                               dz0=5.0, r=1.15, a=(1, 1, 1)),
    # degenerate extents: one free column in x, one free plane in z
    "one_col": lambda: synth.hill(nx=2, ny=70, nz=6, dx=30.0, height=40.0, sigma=200.0,
                                  dz0=5.0, r=1.2, a=(1, 1, 2)),
    "one_plane": lambda: synth.hill(nx=90, ny=33, nz=1, dx=30.0, height=40.0, sigma=200.0,
                                    dz0=5.0, r=1.2, a=(1, 1, 2)),
}


def _pair(wd, p, **kw):
    g = p.to(DEV)
    out = []
    for sm in ("fused", "phased"):
        opt = wd.default_options(coarsest_max_free=60, smoother=sm, **kw)
        out.append(wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt))
    return g, out


@pytest.mark.parametrize("name", list(GRIDS))
def test_fused_equals_phased_every_level(wd, name):
    p = GRIDS[name]()
    g, (cf, cp) = _pair(wd, p)
    rng = np.random.default_rng(11)
    for l in range(cf.num_levels()):
        n1, n2, n3 = cf.level_dims(l)
        x = torch.as_tensor(rng.uniform(-1, 1, (n3, n2, n1)), device=DEV)
        f = torch.as_tensor(rng.uniform(-1, 1, (n3, n2, n1)), device=DEV)
        for sweeps in (1, 2, 3):
            a = wd.wd_smooth(cf, l, x.clone(), f, sweeps=sweeps)
            b = wd.wd_smooth(cp, l, x.clone(), f, sweeps=sweeps)
            torch.cuda.synchronize()
            assert torch.equal(a, b), (name, l, sweeps, (a - b).abs().max().item())
    cf.close()
    cp.close()


@pytest.mark.parametrize("name", ["small", "ragged_a"])
def test_fused_solve_history_identical(wd, name):
    """Same iterates bit for bit; the fused context takes its convergence test
    from the residual variant of each cycle's first sweep (a different
    summation order than the residual pass of the phased context), so the
    residual history agrees to rounding and the cycle counts are equal."""
    p = GRIDS[name]()
    g, (cf, cp) = _pair(wd, p)
    f = wd.wd_rhs(cf, g.u0)
    la, ra = wd.wd_solve(cf, f, rel_tol=1e-10)
    lb, rb = wd.wd_solve(cp, f, rel_tol=1e-10)
    torch.cuda.synchronize()
    assert ra["cycles"] == rb["cycles"]
    # hist is relative to ||f||: rounding of the residual sums is absolute
    assert np.allclose(ra["hist"], rb["hist"], rtol=1e-9, atol=1e-13)
    assert torch.equal(la, lb)
    cf.close()
    cp.close()


@pytest.mark.parametrize("name", ["small", "ragged_a", "one_plane", "thin"])
def test_lagged_residual_matches_vcycle_residuals(wd, name):
    """The residuals wd_solve reads from the first sweep of each cycle (fused
    RES variant) against the residual pass after each wd_vcycle: the same
    iterates, so the same relative residuals to rounding; graph replay and
    direct launches give identical histories and iterates."""
    p = GRIDS[name]()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=60))
    nog = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=60, use_graph=0))
    f = wd.wd_rhs(ctx, g.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
    lam2, rep2 = wd.wd_solve(nog, f, rel_tol=1e-10)
    assert rep["cycles"] == rep2["cycles"] and rep["hist"] == rep2["hist"]
    assert torch.equal(lam, lam2)
    x = torch.zeros_like(f)
    hist = [1.0]
    for _ in range(rep["cycles"]):
        hist.append(wd.wd_vcycle(ctx, x, f))
    assert torch.equal(x, lam)
    assert np.allclose(rep["hist"], hist, rtol=1e-9, atol=1e-13), (rep["hist"], hist)
    ctx.close()
    nog.close()


@pytest.mark.parametrize("use_graph", [1, 0])
def test_lagged_residual_warm_start_and_caps(wd, use_graph):
    """Warm start from the converged iterate: the first sweep's residual passes
    the test, the sweep is dropped and lambda comes back unchanged (0 cycles);
    a cycle cap stops with WD_E_NOCONV after exactly max_cycles cycles, its
    last residual from the residual pass; a second solve on the same context
    repeats the first bit for bit (graph state restored)."""
    p = GRIDS["ragged_a"]()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a,
                         wd.default_options(coarsest_max_free=60, use_graph=use_graph))
    f = wd.wd_rhs(ctx, g.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-9)
    lam_b, rep_b = wd.wd_solve(ctx, f, rel_tol=1e-9)
    assert torch.equal(lam, lam_b) and rep["hist"] == rep_b["hist"]
    lam_w, rep_w = wd.wd_solve(ctx, f, lam0=lam, rel_tol=1e-9)
    assert rep_w["cycles"] == 0 and torch.equal(lam_w, lam)
    assert rep_w["rel_res0"] == pytest.approx(rep["rel_res_final"], rel=1e-3, abs=1e-13)
    # one more cycle from the converged iterate when the tolerance is tighter
    lam_t, rep_t = wd.wd_solve(ctx, f, lam0=lam, rel_tol=rep["rel_res_final"] * 0.5)
    x = lam.clone()
    r1 = wd.wd_vcycle(ctx, x, f)
    assert rep_t["cycles"] >= 1
    if rep_t["cycles"] == 1:
        assert torch.equal(lam_t, x) and rep_t["hist"][1] == pytest.approx(r1, rel=1e-3, abs=1e-13)
    capped = wd.default_options(coarsest_max_free=60, use_graph=use_graph, max_cycles=3)
    c2 = wd.wd_assemble(g.X, g.Y, g.Z, p.a, capped)
    lam_c, rep_c = wd.wd_solve(c2, f, rel_tol=1e-14, raise_on_noconv=False)
    assert rep_c["cycles"] == 3 and not rep_c["converged"]
    x = torch.zeros_like(f)
    for _ in range(3):
        rc = wd.wd_vcycle(c2, x, f)
    assert torch.equal(lam_c, x)
    assert rep_c["rel_res_final"] == pytest.approx(rc, rel=1e-9, abs=1e-13)
    ctx.close()
    c2.close()


def test_fused_sweep_matches_oracle_small(wd):
    """One fused sweep on the fine level of Small against the oracle's GS
    sweep (<= 1e-11 relative max; the orders differ only by FMA contraction)."""
    p = synth.small()
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(smoother="fused"))
    mg = oracle.MG(X, Y, Z, p.a)
    rng = np.random.default_rng(5)
    s = mg.shape(0)
    x = rng.uniform(-1, 1, s) * free_mask(s)
    f = rng.uniform(-1, 1, s) * free_mask(s)
    got = wd.wd_smooth(ctx, 0, torch.as_tensor(x, device=DEV), torch.as_tensor(f, device=DEV),
                       sweeps=2).cpu().numpy()
    ref = mg.gs(0, mg.gs(0, x, f), f)
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-11
    ctx.close()


ZMERGE = {
    # fine vertical spacing against the horizontal one: the planner merges
    # layers after the first horizontal coarsenings (non-identity z maps)
    "zmerge": lambda: synth.hill(nx=120, ny=97, nz=12, dx=15.0, height=60.0, sigma=400.0,
                                 dz0=3.0, r=1.3, a=(1, 1, 1)),
}


@pytest.mark.parametrize("name", ["small", "ragged_a", "ragged_b", "zmerge"])
def test_galerkin_unrolled_path_bitwise(wd, name, monkeypatch):
    """The unrolled Galerkin paths (regular interior columns; identity z map,
    or layers merged with the z pairs built at run time) perform the generic
    kernel's products and sums in the same order: the coarse operators must
    be bit-for-bit those of the generic path."""
    p = (GRIDS.get(name) or ZMERGE[name])()
    g = p.to(DEV)
    opt = wd.default_options(coarsest_max_free=60)
    fast = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    monkeypatch.setenv("WD_GALERKIN_GENERIC", "1")
    gen = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    monkeypatch.delenv("WD_GALERKIN_GENERIC")
    assert fast.num_levels() == gen.num_levels()
    if name in ZMERGE:
        n3s = [fast.level_dims(l)[2] for l in range(fast.num_levels())]
        assert any(b < a for a, b in zip(n3s, n3s[1:])), n3s
    for l in range(1, fast.num_levels()):
        a = wd.wd_get_stencil(fast, l)
        b = wd.wd_get_stencil(gen, l)
        torch.cuda.synchronize()
        assert torch.equal(a, b), (name, l, (a - b).abs().max().item())
    fast.close()
    gen.close()


@pytest.mark.parametrize("name", ["tiny", "small", "ragged_a", "thin"])
def test_line_relaxation_matches_oracle(wd, name):
    """Vertical line relaxation: one GPU sweep on every level
    against the oracle's Thomas-algorithm sweep (<= 1e-11 relative max)."""
    p = GRIDS[name]()
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=60,
                                                                 smoother="line"))
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=60, smoother="line")
    assert ctx.num_levels() == mg.nlev
    rng = np.random.default_rng(9)
    for l in range(mg.nlev):
        s = mg.shape(l)
        x = rng.uniform(-1, 1, s) * free_mask(s)
        f = rng.uniform(-1, 1, s) * free_mask(s)
        got = wd.wd_smooth(ctx, l, torch.as_tensor(x, device=DEV), torch.as_tensor(f, device=DEV),
                           sweeps=1).cpu().numpy()
        ref = mg.gs(l, x, f)
        assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max(), (name, l)
    ctx.close()


@pytest.mark.parametrize("name", ["small", "ragged_a"])
def test_line_relaxation_solve_parity(wd, name):
    """Solves with the line smoother on both sides: lambda within 1e-8
    relative l2 at rel. residual 1e-10, convergence factor within 10 %."""
    p = GRIDS[name]()
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=60,
                                                                 smoother="line"))
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=60, smoother="line")
    f = oracle.rhs(X, Y, Z, u0)
    lam, rep = wd.wd_solve(ctx, torch.as_tensor(f, device=DEV), rel_tol=1e-10)
    lo, ro = mg.solve(f, tol=1e-10)
    lam = lam.cpu().numpy()
    assert np.linalg.norm(lam - lo) <= 1e-8 * np.linalg.norm(lo)
    assert abs(rep["rate"] - ro["rate"]) <= 0.1 * ro["rate"], (rep["rate"], ro["rate"])
    ctx.close()


@pytest.mark.parametrize("nx,ny", [(64, 8), (65, 9), (66, 10), (127, 15), (128, 16), (129, 17),
                                   (63, 7), (62, 23)])
def test_fused_tile_edges(wd, nx, ny):
    """Grids whose node counts sit on, just below and just above the fused
    sweep's 64 x 8 tile boundaries: fused == phased bit for bit on the fine
    level (two sweeps, ping-pong both ways)."""
    p = synth.hill(nx=nx, ny=ny, nz=5, dx=30.0, height=60.0, sigma=300.0, dz0=6.0, r=1.2,
                   a=(1, 1, 4))
    g, (cf, cp) = _pair(wd, p)
    rng = np.random.default_rng(nx * 100 + ny)
    n1, n2, n3 = cf.level_dims(0)
    x = torch.as_tensor(rng.uniform(-1, 1, (n3, n2, n1)), device=DEV)
    f = torch.as_tensor(rng.uniform(-1, 1, (n3, n2, n1)), device=DEV)
    a = wd.wd_smooth(cf, 0, x.clone(), f, sweeps=2)
    b = wd.wd_smooth(cp, 0, x.clone(), f, sweeps=2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    cf.close()
    cp.close()

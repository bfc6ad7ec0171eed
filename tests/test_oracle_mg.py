"""Pins of the oracle's multigrid (Sec. 3): planner hand
traces, dense P / P^T, dense Galerkin P^T K P, dense Gauss-Seidel, dense
two-grid cycle, direct solves, fast diagonalisation, and the paper's
convergence anchors."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from brute import (fast_diag_solve, free_mask, gs_dense, gs_order, line_dense, prolong_dense)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _np(p):
    return p.numpy()


# --------------------------------------------------------------- planner
def test_planner_hand_traces():
    for case in GOLD["planner_traces"]["cases"]:
        for rule in case["rules"]:
            r = oracle.plan_level(case["h1"], case["h3"], case["a"], rule)
            assert r["horizontal"] == case["horizontal"], (case, rule)
            assert r["kept"] == case["kept"], (case, rule, r)


def test_planner_coupling_reading_a3():
    """Reading C1: under Eq. (4) a3 = 10 weakens vertical coupling (c3 =
    a3^-2), so uniform h with a3 = 10 coarsens horizontally only; the printed
    ratio (VERBATIM) coarsens vertically only."""
    for rule in ("coupling_cur", "coupling_paper"):
        r = oracle.plan_level(1.0, [1, 1, 1, 1], (1, 1, 10), rule)
        assert r["horizontal"] and r["kept"] == [0, 1, 2, 3, 4]
    r = oracle.plan_level(1.0, [1, 1, 1, 1], (1, 1, 10), "verbatim")
    assert not r["horizontal"] and r["kept"] == [0, 2, 4]


def test_planner_c1b_current_vs_coarsened_h1():
    """C1b: the vertical test uses the current h1 (CUR) or the coarsened 2*h1
    (PAPER).  h1 = 1, h3 = [2, 2, 2, 2]: rho = 2 < 3 merges under CUR, while
    2/(2) = 1 also merges under PAPER; h3 = [4, ...]: CUR keeps (4 >= 3),
    PAPER merges (2 < 3)."""
    r = oracle.plan_level(1.0, [4, 4, 4, 4], (1, 1, 1), "coupling_cur")
    assert r["horizontal"] and r["kept"] == [0, 1, 2, 3, 4]
    r = oracle.plan_level(1.0, [4, 4, 4, 4], (1, 1, 1), "coupling_paper")
    assert r["horizontal"] and r["kept"] == [0, 2, 4]
    r = oracle.plan_level(1.0, [4, 4, 4, 4, 4], (1, 1, 1), "coupling_paper")
    assert r["kept"] == [0, 2, 4, 5] and list(r["h3"]) == [8, 8, 4]


def test_hierarchy_uniform_33():
    """33x33x17-node uniform grid, a3 = 1, threshold 200 -> levels
    shrink ~8x, >= 3 levels."""
    p = synth.box(32, 32, 16)
    mg = oracle.MG(*_np(p)[:3], p.a, coarsest_max_free=200)
    assert mg.dims == [(33, 33, 17), (17, 17, 9), (9, 9, 5)]
    for pl in mg.plans:
        assert pl["horizontal"]


# --------------------------------------------------------------- transfer
def _small_hierarchy(a=(1, 1, 1), cmax=40):
    p = synth.hill(nx=10, ny=8, nz=6, dx=50.0, height=80.0, sigma=150.0, dz0=10.0, r=1.2,
                   a=a)
    X, Y, Z, _ = _np(p)
    return p, oracle.MG(X, Y, Z, a, coarsest_max_free=cmax)


def test_prolong_restrict_dense():
    """P x_c and P^T r equal the dense index-space trilinear P;
    P 1 = 1 on free nodes; <P x, y> = <x, P^T y>."""
    p, mg = _small_hierarchy()
    assert mg.nlev >= 2
    rng = np.random.default_rng(0)
    for l in range(mg.nlev - 1):
        fs, cs = mg.shape(l), mg.shape(l + 1)
        P, cshape = prolong_dense(fs, mg.plans[l]["horizontal"], mg.plans[l]["kept"])
        assert cshape == cs
        fm, cm = free_mask(fs).ravel(), free_mask(cs).ravel()
        xc = rng.uniform(-1, 1, cs) * free_mask(cs)
        x0 = rng.uniform(-1, 1, fs) * free_mask(fs)
        got = mg.prolong(l, xc, x0)
        want = (x0.ravel() + (P @ xc.ravel()) * fm).reshape(fs)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)
        ones = free_mask(cs).astype(float)
        pu = mg.prolong(l, ones, np.zeros(fs))
        # P 1 = 1 away from the coarse Dirichlet nodes' support
        assert np.allclose(pu.ravel()[fm & ((P[:, ~cm].sum(1)) == 0)], 1.0)
        r = rng.uniform(-1, 1, fs) * free_mask(fs)
        fc = mg.restrict(l, r)
        want = (P.T @ r.ravel()) * cm
        np.testing.assert_allclose(fc.ravel(), want, rtol=0, atol=1e-14)
        lhs = np.dot(mg.prolong(l, xc, np.zeros(fs)).ravel(), r.ravel())
        rhs = np.dot(xc.ravel(), fc.ravel())
        assert abs(lhs - rhs) <= 1e-13 * (abs(lhs) + 1)


def test_restrict_constant_gives_8():
    """Full coarsening, constant fine field 1 -> 8 at an interior coarse node
    (1 + 6/2 + 12/4 + 8/8)."""
    p = synth.box(8, 8, 8)
    mg = oracle.MG(*_np(p)[:3], p.a, coarsest_max_free=30)
    fc = mg.restrict(0, free_mask(mg.shape(0)).astype(float))
    assert fc[1, 2, 2] == 8.0


def test_galerkin_dense_all_levels():
    """K_{l+1} = P^T K_l P on the free block (Eq. (7), C11), dense brute force."""
    p, mg = _small_hierarchy(a=(1, 1, 3), cmax=20)
    assert mg.nlev >= 3
    for l in range(mg.nlev - 1):
        fs, cs = mg.shape(l), mg.shape(l + 1)
        P, _ = prolong_dense(fs, mg.plans[l]["horizontal"], mg.plans[l]["kept"])
        fm, cm = free_mask(fs).ravel(), free_mask(cs).ravel()
        A = oracle.stencil_to_dense(mg.K(l))[np.ix_(fm, fm)]
        Pf = P[np.ix_(fm, cm)]
        want = Pf.T @ A @ Pf
        got = oracle.stencil_to_dense(mg.K(l + 1))[np.ix_(cm, cm)]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("plan", ["full", "horizontal", "vertical"])
def test_galerkin_nested_box_equals_rediscretisation(plan):
    """Uniform box, nested Q1 spaces: P^T K P = K assembled directly on the
    coarse box, for full and semi-coarsening."""
    n = 8
    p = synth.box(n, n, n, dx=1.0, dy=1.0, dz=1.0)
    X, Y, Z, _ = _np(p)
    a = (1.0, 1.0, 2.0)
    K = oracle.assemble(X, Y, Z, a)
    hflag = plan in ("full", "horizontal")
    kept = list(range(0, n + 1, 2)) if plan in ("full", "vertical") else list(range(n + 1))
    Kc = oracle.galerkin(K, hflag, kept)
    hc = 2.0 if hflag else 1.0
    zc = 2.0 if plan != "horizontal" else 1.0
    nc = n // 2 if hflag else n
    nzc = len(kept) - 1
    q = synth.box(nc, nc, nzc, dx=hc, dy=hc, dz=zc)
    Kd = oracle.assemble(*_np(q)[:3], a)
    cm = free_mask(Kd.shape[:3])
    np.testing.assert_allclose(Kc[cm], Kd[cm], rtol=0, atol=1e-13 * np.abs(Kd).max())


# --------------------------------------------------------------- smoother
def test_gs_sweep_is_dense_triangular_solve():
    """4-colour bottom-up column GS == standard GS in the order (colour,
    column, k) == (D + L)^{-1}(f - U x)."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    K = oracle.assemble(X, Y, Z, (1, 1, 4))
    A = oracle.stencil_to_dense(K)
    f = oracle.rhs(X, Y, Z, u0)
    x0 = synth.random_lambda(p, 1).numpy()
    got = oracle.gs_sweep(K, x0, f)
    want = gs_dense(A, f, x0, gs_order(X.shape))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())
    # fixed point and K-norm monotonicity
    m = free_mask(X.shape).ravel()
    xs = np.zeros(m.size)
    xs[m] = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    xs = xs.reshape(X.shape)
    np.testing.assert_allclose(oracle.gs_sweep(K, xs, f), xs, atol=1e-12 * np.abs(xs).max())
    x = x0
    e_prev = np.inf
    for _ in range(4):
        d = (x - xs).ravel()
        e = d @ A @ d
        assert e <= e_prev
        e_prev = e
        x = oracle.gs_sweep(K, x, f)


def test_gs_single_free_node_exact():
    p = synth.box(2, 2, 1)
    X, Y, Z, _ = _np(p)
    K = oracle.assemble(X, Y, Z, (1, 1, 1))
    f = np.zeros(X.shape)
    f[0, 1, 1] = 3.0
    x = oracle.gs_sweep(K, np.zeros(X.shape), f)
    assert x[0, 1, 1] == 3.0 / K[0, 1, 1, 13]


def test_line_sweep_is_dense_block_gs():
    """Vertical line relaxation == block GS over free columns
    in the colour order, each column block solved densely (numpy), on Tiny
    with a3 = 4; plus the fixed point and K-norm monotonicity."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    K = oracle.assemble(X, Y, Z, (1, 1, 4))
    A = oracle.stencil_to_dense(K)
    f = oracle.rhs(X, Y, Z, u0)
    x0 = synth.random_lambda(p, 1).numpy()
    got = oracle.line_sweep(K, x0, f)
    want = line_dense(A, f, x0, X.shape)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * np.abs(want).max())
    m = free_mask(X.shape).ravel()
    xs = np.zeros(m.size)
    xs[m] = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    xs = xs.reshape(X.shape)
    np.testing.assert_allclose(oracle.line_sweep(K, xs, f), xs, atol=1e-12 * np.abs(xs).max())
    x = x0
    e_prev = np.inf
    for _ in range(4):
        d = (x - xs).ravel()
        e = d @ A @ d
        assert e <= e_prev
        e_prev = e
        x = oracle.line_sweep(K, x, f)


def test_line_single_column_exact():
    """One free column (2x2 elements in x-y): one line sweep solves K x = f
    exactly (the column block is the whole free system)."""
    p = synth.box(2, 2, 6, dz=np.array([1.0, 2.0, 3.0, 1.0, 2.0, 4.0]))
    X, Y, Z, _ = _np(p)
    K = oracle.assemble(X, Y, Z, (1, 1, 3))
    A = oracle.stencil_to_dense(K)
    m = free_mask(X.shape).ravel()
    rng = np.random.default_rng(3)
    f = rng.standard_normal(X.shape) * free_mask(X.shape)
    x = oracle.line_sweep(K, np.zeros(X.shape), f)
    xs = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    np.testing.assert_allclose(x.ravel()[m], xs, rtol=0, atol=1e-13 * np.abs(xs).max())


@pytest.mark.parametrize("a3", [1, 10])
def test_mg_line_smoother_matches_dense_direct_tiny(a3):
    """The V-cycle with line relaxation converges to the dense direct
    solution (1e-8 relative l2 at rel. residual 1e-10)."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    a = (1, 1, a3)
    f = oracle.rhs(X, Y, Z, u0)
    mg = oracle.MG(X, Y, Z, a, coarsest_max_free=100, smoother="line")
    lam, rep = mg.solve(f, tol=1e-10)
    assert rep["status"] == 0 and rep["cycles"] <= 30
    A = oracle.stencil_to_dense(oracle.assemble(X, Y, Z, a))
    m = free_mask(X.shape).ravel()
    xs = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    assert np.linalg.norm(lam.ravel()[m] - xs) <= 1e-8 * np.linalg.norm(xs)


# --------------------------------------------------------------- cycles
def test_two_grid_cycle_dense():
    """Two-level V-cycle = S_post o (I + P Kc^{-1} P^T (f - K .)) o S_pre with
    dense matrices."""
    p, mg = _small_hierarchy(a=(1, 1, 1), cmax=200)
    assert mg.nlev == 2 and mg.coarse_direct
    fs, cs = mg.shape(0), mg.shape(1)
    X, Y, Z, u0 = _np(p)
    f = oracle.rhs(X, Y, Z, u0)
    A = oracle.stencil_to_dense(mg.K(0))
    fm, cm = free_mask(fs).ravel(), free_mask(cs).ravel()
    P, _ = prolong_dense(fs, mg.plans[0]["horizontal"], mg.plans[0]["kept"])
    Pf = P[np.ix_(fm, cm)]
    Kc = Pf.T @ A[np.ix_(fm, fm)] @ Pf
    order = gs_order(fs)
    x = synth.random_lambda(p, 2).numpy()
    got = mg.vcycle(x, f)
    for _ in range(2):
        x = gs_dense(A, f, x, order)
    r = (f.ravel() - A @ x.ravel())[fm]
    xc = np.linalg.solve(Kc, Pf.T @ r)
    xv = x.ravel().copy()
    xv[fm] += Pf @ xc
    x = xv.reshape(fs)
    for _ in range(2):
        x = gs_dense(A, f, x, order)
    np.testing.assert_allclose(got, x, rtol=0, atol=1e-12 * np.abs(x).max())


def test_zero_rhs_fixed_point():
    p, mg = _small_hierarchy(cmax=20)
    z = np.zeros(mg.shape(0))
    assert not mg.vcycle(z, z).any()


def test_coarse_direct_solve_dense():
    p, mg = _small_hierarchy(cmax=200)
    cs = mg.shape(mg.nlev - 1)
    cm = free_mask(cs).ravel()
    rng = np.random.default_rng(3)
    fc = rng.normal(size=cs) * free_mask(cs)
    x = mg.coarse_solve(fc)
    A = oracle.stencil_to_dense(mg.K(mg.nlev - 1))[np.ix_(cm, cm)]
    want = np.linalg.solve(A, fc.ravel()[cm])
    np.testing.assert_allclose(x.ravel()[cm], want, rtol=0, atol=1e-11 * np.abs(want).max())


@pytest.mark.parametrize("a", [(1, 1, 1), (1, 1, 10)])
def test_mg_solve_matches_dense_direct_tiny(a):
    """S:366 / S:540: multigrid solution = dense direct solve <= 1e-8 rel l2."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    mg = oracle.MG(X, Y, Z, a, coarsest_max_free=60)
    assert mg.nlev >= 3
    f = oracle.rhs(X, Y, Z, u0)
    lam, rep = mg.solve(f, tol=1e-10)
    assert rep["status"] == 0
    A = oracle.stencil_to_dense(mg.K(0))
    m = free_mask(X.shape).ravel()
    ls = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    err = np.linalg.norm(lam.ravel()[m] - ls) / np.linalg.norm(ls)
    assert err <= 1e-8
    # warm start from the solution: <= 1 cycle
    lam2, rep2 = mg.solve(f, lam0=lam, tol=1e-10)
    assert rep2["cycles"] <= 1


def test_fast_diagonalisation_flat_small():
    """Flat, stretched Small variant: lambda* by fast diagonalisation (1-D
    generalised eigenproblems, independent of the oracle's assembly) vs the
    oracle's MG solve <= 1e-8 relative l2."""
    p = synth.flat_variant(synth.small())
    X, Y, Z, u0 = _np(p)
    a = (1.0, 1.0, 10.0)
    c = 1 / np.array(a) ** 2
    f = oracle.rhs(X, Y, Z, u0)
    hz = np.diff(Z[:, 0, 0])
    ref = fast_diag_solve(np.full(128, 50.0), np.full(128, 50.0), hz, c, f)
    mg = oracle.MG(X, Y, Z, a)
    lam, rep = mg.solve(f, tol=1e-11, max_cycles=60)
    assert rep["status"] == 0
    err = np.linalg.norm(lam - ref) / np.linalg.norm(ref)
    assert err <= 1e-8, err


# --------------------------------------------------------------- anchors
def test_rate_regular_grid_anchor():
    """P:169-172 (~0.1 for Poisson on a regular grid with 4-5 GS sweeps),
    relaxed to <= 0.15 as in S:538: 32x32x16 uniform box, 2+2 smoothing,
    geometric mean over cycles 2..8."""
    p = synth.box(32, 32, 16)
    X, Y, Z, _ = _np(p)
    rng = np.random.default_rng(0)
    f = rng.standard_normal(X.shape) * free_mask(X.shape)
    mg = oracle.MG(X, Y, Z, (1, 1, 1), coarsest_max_free=200)
    _, rep = mg.solve(f, tol=1e-30, max_cycles=8)
    assert rep["cycles"] == 8
    assert rep["rate"] <= 0.15


@pytest.mark.parametrize("a3", [1, 10, 100])
def test_rate_semicoarsening_hill_anchor(a3):
    """P:200-202 ("up to about 0.28 with four smoothing steps"), relaxed to
    <= 0.35 as in S:539: 64x64x16 Gaussian hill (height 100 m, sigma 500 m,
    dx 50 m), stretch 1.3, a3 in {1, 10, 100}."""
    p = synth.hill(height=100.0, a=(1, 1, a3))
    X, Y, Z, _ = _np(p)
    rng = np.random.default_rng(0)
    f = rng.standard_normal(X.shape) * free_mask(X.shape)
    mg = oracle.MG(X, Y, Z, p.a)
    _, rep = mg.solve(f, tol=1e-30, max_cycles=10)
    assert rep["rate"] <= 0.35, rep["rate"]
    # the f1 line-relaxation smoother meets the same anchor (measured 0.22 / 0.11 / 0.28)
    mg = oracle.MG(X, Y, Z, p.a, smoother="line")
    _, rep = mg.solve(f, tol=1e-30, max_cycles=10)
    assert rep["rate"] <= 0.35, rep["rate"]

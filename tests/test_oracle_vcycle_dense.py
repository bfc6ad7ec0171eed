"""The oracle's whole multi-level V-cycle against a dense, recursive
re-implementation written from the paper's Eq. (7) and P:128-158 with numpy
matrices only (tests/brute.py: dense index-space P, dense Gauss-Seidel as a
triangular solve in the colour/column/k order, dense column-block line
relaxation, dense Galerkin P_F^T K_FF P_F, numpy solves):

    V_l(x, f) = S_post^2( x' + P_l V_{l+1}(0, P_l^T (f - K_l x')) ),  x' = S_pre^2(x)
    V_L(0, f) = K_L^{-1} f   (or 50 sweeps of the smoother from 0, reading C8).

Equal cycles make equal convergence factors, so this pins the oracle's rate
(C10) on hierarchies of 3-4 levels beyond the paper's two anchors -- the part
of the oracle round 1 had to leave "parity unpinned".  The dense cycle shares
nothing with orc.c but the stored fine-level stencil and the plan (both pinned
elsewhere: test_oracle_assembly.py, test_oracle_mg.py planner traces).
"""
import numpy as np
import pytest

import oracle
import synth
from brute import free_mask, gs_dense, gs_order, line_dense, prolong_dense


def _dense_hierarchy(mg):
    """Full-size dense matrices per level with only the free block set."""
    levels = []
    K0 = oracle.stencil_to_dense(mg.K(0))
    m0 = free_mask(mg.shape(0)).ravel()
    A = np.zeros_like(K0)
    A[np.ix_(m0, m0)] = K0[np.ix_(m0, m0)]
    levels.append(A)
    Ps = []
    for l in range(mg.nlev - 1):
        fs, cs = mg.shape(l), mg.shape(l + 1)
        P, dims = prolong_dense(fs, mg.plans[l]["horizontal"], mg.plans[l]["kept"])
        assert tuple(dims) == tuple(cs)
        fm, cm = free_mask(fs).ravel(), free_mask(cs).ravel()
        Pf = np.zeros_like(P)
        Pf[np.ix_(fm, cm)] = P[np.ix_(fm, cm)]
        Ps.append(Pf)
        levels.append(Pf.T @ levels[-1] @ Pf)
    return levels, Ps


def _dense_vcycle(mg, levels, Ps, l, x, f, smoothers, coarse_direct, coarse_iters=50):
    shape = mg.shape(l)
    A = levels[l]
    m = free_mask(shape).ravel()

    def sweep(v):
        if smoothers[l] == "line":
            return line_dense(A, f, v, shape)
        return gs_dense(A, f, v, gs_order(shape))

    if l == mg.nlev - 1:
        if coarse_direct:
            out = np.zeros(A.shape[0])
            out[m] = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
            return out.reshape(shape)
        v = np.zeros(shape)
        for _ in range(coarse_iters):
            v = sweep(v)
        return v
    for _ in range(2):
        x = sweep(x)
    r = f.ravel() - A @ x.ravel()
    r[~m] = 0.0
    fc = (Ps[l].T @ r).reshape(mg.shape(l + 1))
    xc = _dense_vcycle(mg, levels, Ps, l + 1, np.zeros(mg.shape(l + 1)), fc, smoothers,
                       coarse_direct, coarse_iters)
    x = (x.ravel() + Ps[l] @ xc.ravel()).reshape(shape)
    for _ in range(2):
        x = sweep(x)
    return x


CASES = {
    # name: (a, coarsest_max_free, smoother, line_from_level)
    "gs_direct": ((1, 1, 1), 8, "gs", -1),
    "gs_a3_direct": ((1, 1, 10), 40, "gs", -1),
    "gs_iterative_coarsest": ((1, 1, 1), 0, "gs", -1),
    "line": ((1, 1, 10), 40, "line", -1),
    "per_level": ((1, 1, 10), 40, "gs", 1),
}


@pytest.mark.parametrize("case", list(CASES))
def test_multilevel_vcycle_dense(case):
    a, cmax, smoother, lf = CASES[case]
    p = synth.hill(nx=10, ny=8, nz=6, dx=50.0, height=80.0, sigma=150.0, dz0=10.0, r=1.2, a=a)
    X, Y, Z, u0 = p.numpy()
    mg = oracle.MG(X, Y, Z, a, coarsest_max_free=cmax, smoother=smoother, line_from_level=lf)
    assert mg.nlev >= 3
    smoothers = [("line" if (smoother == "line" or (lf >= 0 and l >= lf)) else "gs")
                 for l in range(mg.nlev)]
    levels, Ps = _dense_hierarchy(mg)
    f = oracle.rhs(X, Y, Z, u0)
    x0 = synth.random_lambda(p, 5).numpy()
    got = mg.vcycle(x0, f)
    want = _dense_vcycle(mg, levels, Ps, 0, x0, f, smoothers, mg.coarse_direct)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-11 * np.abs(want).max())
    # residual history of six cycles from zero (the convergence factor, C10)
    fm = free_mask(mg.shape(0)).ravel()
    A0 = levels[0]
    fn = np.linalg.norm(f.ravel()[fm])
    x = np.zeros_like(f)
    hist = [1.0]
    for _ in range(6):
        x = _dense_vcycle(mg, levels, Ps, 0, x, f, smoothers, mg.coarse_direct)
        hist.append(np.linalg.norm((f.ravel() - A0 @ x.ravel())[fm]) / fn)
    _, rep = mg.solve(f, tol=hist[6] * 0.999, max_cycles=6)
    # the two differ by rounding only: ~1e-16 of ||K|| ||x|| in every residual, which
    # is ~1e-8 of a residual that has fallen to ~1e-8 after six fast cycles
    np.testing.assert_allclose(rep["hist"][:7], hist, rtol=1e-6, atol=1e-14)
    rate_dense = (hist[6] / hist[1]) ** (1.0 / 5)
    assert abs(rep["rate"] - rate_dense) <= 1e-6 * rate_dense

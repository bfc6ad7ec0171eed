"""Pins of the oracle's global assembly, RHS and recovery (Eq. (3),
(5)) against closed forms, brute force and exact identities."""
import numpy as np
import pytest

import oracle
import synth
from brute import box_stiffness_dense, free_mask


def _np(p):
    return p.numpy()


@pytest.mark.parametrize("dz,c", [(1.0, (1, 1, 1)), ([1.0, 2.0, 4.0, 3.0], (1, 0.5, 0.01))])
def test_flat_box_kronecker(dz, c):
    """Flat (box) grids, any vertical stretching: assembled K equals the
    Kronecker sum of 1-D stiffness/mass matrices (SURVEY 8(c) pin)."""
    nz = 4
    p = synth.box(5, 4, nz, dx=2.0, dy=3.0, dz=dz)
    X, Y, Z, _ = _np(p)
    a = tuple(1 / np.sqrt(ci) for ci in c)
    K = oracle.assemble(X, Y, Z, a)
    A = oracle.stencil_to_dense(K)
    hz = np.full(nz, dz) if np.isscalar(dz) else np.array(dz)
    ref = box_stiffness_dense(np.full(5, 2.0), np.full(4, 3.0), hz, c)
    np.testing.assert_allclose(A, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_uniform_cube_interior_stencil():
    """Uniform cube h: interior stencil centre 8h/3, face 0, edge -h/6, corner -h/12."""
    h = 2.5
    p = synth.box(4, 4, 4, dx=h, dy=h, dz=h)
    K = oracle.assemble(*_np(p)[:3], (1, 1, 1))
    row = K[2, 2, 2]
    for o in range(27):
        d = (o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1)
        nz_ = sum(abs(v) for v in d)
        want = {0: 8 * h / 3, 1: 0.0, 2: -h / 6, 3: -h / 12}[nz_]
        assert abs(row[o] - want) <= 1e-14 * h


def test_symmetry_rowsum_psd_tiny():
    p = synth.tiny()
    X, Y, Z, _ = _np(p)
    K = oracle.assemble(X, Y, Z, (1, 1, 3))
    A = oracle.stencil_to_dense(K)
    assert np.array_equal(A, A.T)                             # bitwise
    np.testing.assert_allclose(A.sum(1), 0, atol=1e-12 * np.abs(A).max())
    m = free_mask(X.shape).ravel()
    w = np.linalg.eigvalsh(A[np.ix_(m, m)])
    assert w[0] > 0


def test_patch_test_and_energy_on_hill():
    """Linear lambda: (K lambda)_p = 0 at nodes away from the boundary (2x2x2
    Gauss is exact for it on trilinear elements), and lambda^T K lambda =
    g^T C g * volume, volume = sum of dx dy mean(dz) over columns."""
    p = synth.tiny()
    X, Y, Z, _ = _np(p)
    a = (1.0, 2.0, 5.0)
    c = 1 / np.array(a) ** 2
    K = oracle.assemble(X, Y, Z, a)
    g = np.array([0.3, -1.2, 0.7])
    lam = g[0] * X + g[1] * Y + g[2] * Z
    A = oracle.stencil_to_dense(K)
    r = (A @ lam.ravel()).reshape(X.shape)
    scale = (np.abs(A) @ np.abs(lam.ravel())).max()
    assert np.abs(r[1:-1, 1:-1, 1:-1]).max() <= 1e-13 * scale
    dz = Z[1:] - Z[:-1]
    vol = (30.0 * 30.0 * 0.25 * (dz[:, :-1, :-1] + dz[:, :-1, 1:] + dz[:, 1:, :-1]
                                 + dz[:, 1:, 1:])).sum()
    e = lam.ravel() @ (A @ lam.ravel())
    assert abs(e - (c * g) @ g * vol) <= 1e-11 * abs(e)


def test_dense_direct_tiny_and_hill_sign():
    """S:424 hill pattern: u0 = (5,0,0), a = 1, exact lambda* by a dense solve;
    lowest-layer w > 0 on the windward slope and < 0 on the lee side."""
    p = synth.tiny()
    X, Y, Z, _ = _np(p)
    u0 = np.zeros((3, 8, 16, 16))
    u0[0] = 5.0
    K = oracle.assemble(X, Y, Z, (1, 1, 1))
    f = oracle.rhs(X, Y, Z, u0)
    A = oracle.stencil_to_dense(K)
    m = free_mask(X.shape).ravel()
    lam = np.zeros(m.size)
    lam[m] = np.linalg.solve(A[np.ix_(m, m)], f.ravel()[m])
    lam = lam.reshape(X.shape)
    u = oracle.recover(X, Y, Z, (1, 1, 1), lam, u0)
    w = u[2, 0]
    assert w[8, 4] > 0.5 and w[8, 11] < -0.5       # j = 8 row through the peak
    assert w[8, 5] > 0 and w[8, 10] < 0


def test_rhs_divergence_free_inputs_flat():
    """Flat box: constant horizontal u0 and the linear divergence-free
    u0 = (x, -y, 0) give f_F = 0 (one-point quadrature is exact there;
    S:182).  u0 must be tangential on Gamma: a vertical component is
    a genuine flux through the free bottom nodes (natural condition of Eq. (4))."""
    p = synth.box(6, 5, 4, dx=2.0, dy=3.0, dz=[1, 2, 3, 4])
    X, Y, Z, _ = _np(p)
    u0 = np.zeros((3, 4, 5, 6))
    u0[0], u0[1] = 3.0, -1.0
    f = oracle.rhs(X, Y, Z, u0)
    assert np.abs(f).max() <= 1e-13 * 3 * 2 * 3 * 4
    xc = 0.5 * (X[:-1, :-1, :-1] + X[:-1, :-1, 1:])
    yc = 0.5 * (Y[:-1, :-1, :-1] + Y[:-1, 1:, :-1])
    u0 = np.stack([xc, -yc, np.zeros_like(xc)])
    f = oracle.rhs(X, Y, Z, u0)
    assert np.abs(f).max() <= 1e-13 * 12 * 24


def test_flat_uniform_wind_identity():
    """Flat + uniform horizontal u0: f_F = 0 -> lambda = 0 -> u = u0."""
    p = synth.flat_variant(synth.tiny())
    X, Y, Z, _ = _np(p)
    u0 = np.zeros((3, 8, 16, 16))
    u0[0], u0[1] = 5.0, -2.0
    f = oracle.rhs(X, Y, Z, u0)
    assert np.abs(f).max() <= 1e-12
    mg = oracle.MG(X, Y, Z, (1, 1, 1))
    lam, rep = mg.solve(f)
    assert np.abs(lam).max() <= 1e-9 * 5.0 * 480.0     # 1e-9 * |u0| * domain
    u = oracle.recover(X, Y, Z, (1, 1, 1), lam, u0)
    np.testing.assert_allclose(u, u0, rtol=0, atol=1e-9 * 5.0)
    lam, rep = mg.solve(np.zeros_like(f))
    assert rep["cycles"] == 0 and not lam.any()


def test_recover_linear_lambda_on_hill():
    """lambda = g.x (nodal interpolation) -> u = u0 + C g in every element,
    exactly up to rounding, on the distorted terrain grid."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    a = (1.0, 2.0, 4.0)
    g = np.array([1.0, 0.5, -2.0])
    lam = g[0] * X + g[1] * Y + g[2] * Z
    u = oracle.recover(X, Y, Z, a, lam, u0)
    want = u0 + (g / np.array(a) ** 2)[:, None, None, None]
    np.testing.assert_allclose(u, want, rtol=0, atol=1e-12 * np.abs(lam).max() / 5)
    u = oracle.recover(X, Y, Z, a, np.zeros_like(X), u0)
    assert np.array_equal(u, u0)


def test_c12_divergence_identity():
    """D1(u_rec) - (K1 - K) lambda = K lambda - f on free nodes (exact
    algebraic identity; reading C12), and f = -D1(u0)."""
    p = synth.tiny()
    X, Y, Z, u0 = _np(p)
    a = (1.0, 1.0, 2.0)
    lam = synth.random_lambda(p, seed=3).numpy()
    K = oracle.assemble(X, Y, Z, a)
    K1 = oracle.assemble_onepoint(X, Y, Z, a)
    f = oracle.rhs(X, Y, Z, u0)
    np.testing.assert_allclose(f, -oracle.d1(X, Y, Z, u0), rtol=0, atol=1e-12 * np.abs(f).max())
    u = oracle.recover(X, Y, Z, a, lam, u0)
    lhs = oracle.d1(X, Y, Z, u) - (oracle.apply(K1, lam) - oracle.apply(K, lam))
    rhs_ = oracle.apply(K, lam) - f
    m = free_mask(X.shape)
    scale = np.abs(oracle.apply(K, lam)).max() + np.abs(f).max()
    np.testing.assert_allclose(lhs[m], rhs_[m], rtol=0, atol=1e-12 * scale)


def test_validate_mesh_reports_lowest_bad_element():
    p = synth.tiny()
    X, Y, Z, _ = _np(p)
    assert oracle.validate_mesh(X, Y, Z)[0] is None
    Z = Z.copy()
    Z[3, 5, 7], Z[4, 5, 7] = Z[4, 5, 7], Z[3, 5, 7]     # swap two levels at node (7,5)
    e, what = oracle.validate_mesh(X, Y, Z)
    # the inverted edge lies in elements (6..7, 4..5, 3); lowest is (6,4,3)
    assert e == (3 * 16 + 4) * 16 + 6 and what == 0


def test_stencil_asymmetry_helper():
    """The shifted-array symmetry check used on large GPU stencils agrees with
    the dense check: 0 on the oracle's assembled K, > 0 once perturbed."""
    from brute import stencil_asymmetry
    p = synth.tiny()
    K = oracle.assemble(*_np(p)[:3], (1, 1, 2))
    assert stencil_asymmetry(K) == 0.0
    K[3, 4, 5, 14] += 1e-9
    assert stencil_asymmetry(K) > 0

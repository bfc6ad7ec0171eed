"""Pins of the oracle's steps either side of the path: the
terrain-following mesh generator (reading C13) and the coarse-wind
interpolation to element centres.  Closed forms and invariants:
SPEC's build_mesh examples, translation invariance, exact bottom/top, the
synthetic-input recipe (an independent torch implementation), and exact
reproduction of trilinear (linear in x, y, height) fields."""
import numpy as np
import pytest

import oracle
import synth


def test_build_mesh_flat_uniform_spec_example():
    """SPEC build_mesh: flat terrain, uniform levels, H = 10, n3 = 2 layers
    -> Z in {0, 5, 10} at every column."""
    zs = np.zeros((4, 5))
    X, Y, Z = oracle.build_mesh(zs, 0.0, 0.0, 100.0, 50.0, [0.0, 5.0, 10.0], 10.0)
    assert Z.shape == (3, 4, 5)
    for k, z in enumerate([0.0, 5.0, 10.0]):
        assert np.all(Z[k] == z)
    np.testing.assert_array_equal(X[1, 2], 100.0 * np.arange(5))
    np.testing.assert_array_equal(Y[2, :, 3], 50.0 * np.arange(4))


def test_build_mesh_translation_and_bounds():
    rng = np.random.default_rng(4)
    zeta = np.concatenate([[0.0], np.cumsum(10.0 * 1.2 ** np.arange(6))])
    T = zeta[-1]
    zs = rng.uniform(0, 300, (7, 9))
    H = zs.max() + T
    X, Y, Z = oracle.build_mesh(zs, 10.0, -5.0, 30.0, 30.0, zeta, H)
    np.testing.assert_array_equal(Z[0], zs)                       # bottom = terrain
    np.testing.assert_allclose(Z[-1], H, rtol=0, atol=1e-12 * H)  # flat top
    assert np.all(np.diff(Z, axis=0) > 0)                          # no inverted cells
    assert oracle.validate_mesh(X, Y, Z)[0] is None                # every detJ > 0
    # the highest column carries the levels zeta exactly (reading C13)
    jj, ii = np.unravel_index(np.argmax(zs), zs.shape)
    np.testing.assert_allclose(Z[:, jj, ii] - zs[jj, ii], zeta, rtol=0, atol=1e-12 * H)
    # constant terrain c with H = c + T is the flat mesh shifted by c
    c = 123.0
    _, _, Zc = oracle.build_mesh(np.full((3, 4), c), 0, 0, 1, 1, zeta, c + T)
    _, _, Z0 = oracle.build_mesh(np.zeros((3, 4)), 0, 0, 1, 1, zeta, T)
    np.testing.assert_allclose(Zc, Z0 + c, rtol=0, atol=1e-12 * (c + T))


def test_build_mesh_matches_synthetic_recipe():
    """The Tiny config's mesh (synth, torch implementation of the same recipe)
    is reproduced from its terrain and levels."""
    p = synth.tiny()
    X, Y, Z, _ = p.numpy()
    zs = Z[0]
    zeta = Z[:, np.unravel_index(np.argmax(zs), zs.shape)[0],
             np.unravel_index(np.argmax(zs), zs.shape)[1]] - zs.max()
    H = Z[-1].max()
    Xo, Yo, Zo = oracle.build_mesh(zs, 0.0, 0.0, X[0, 0, 1], Y[0, 1, 0], zeta, H)
    np.testing.assert_allclose(Xo, X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(Yo, Y, rtol=0, atol=1e-12)
    np.testing.assert_allclose(Zo, Z, rtol=0, atol=1e-11 * H)


def test_build_mesh_rejects_top_below_terrain():
    zs = np.zeros((3, 3))
    zs[1, 2] = 50.0
    with pytest.raises(ValueError, match="column 5"):
        oracle.build_mesh(zs, 0, 0, 1, 1, [0.0, 10.0, 20.0], 40.0)


def _hill_mesh(nx=12, ny=10, nz=6):
    p = synth.hill(nx=nx, ny=ny, nz=nz, dx=100.0, height=150.0, sigma=300.0, dz0=10.0, r=1.3)
    return p.numpy()[:3]


def _centres(X, Y, Z):
    def m8(A):
        return 0.125 * (A[:-1, :-1, :-1] + A[:-1, :-1, 1:] + A[:-1, 1:, :-1] + A[:-1, 1:, 1:]
                        + A[1:, :-1, :-1] + A[1:, :-1, 1:] + A[1:, 1:, :-1] + A[1:, 1:, 1:])
    zb = 0.25 * (Z[0, :-1, :-1] + Z[0, :-1, 1:] + Z[0, 1:, :-1] + Z[0, 1:, 1:])
    return m8(X), m8(Y), m8(Z) - zb[None]


def test_interp_reproduces_trilinear_fields():
    """A field linear in (x, y, height above ground) sampled on the coarse grid
    is reproduced exactly at every element centre inside the coarse grid."""
    X, Y, Z = _hill_mesh()
    xe, ye, he = _centres(X, Y, Z)
    hc = np.array([0.5, 3.0, 20.0, 60.0, 400.0, 2000.0])
    nxc, nyc = 5, 4
    xc0, yc0, DXc, DYc = -150.0, -80.0, 400.0, 420.0
    xs = xc0 + DXc * np.arange(nxc)
    ys = yc0 + DYc * np.arange(nyc)
    coef = np.array([[5.0, 0.002, -0.001, 0.01], [-1.0, 0.0005, 0.003, -0.002],
                     [0.2, 0.0, 0.0001, 0.0003]])
    uc = np.empty((3, hc.size, nyc, nxc))
    for m in range(3):
        uc[m] = (coef[m, 0] + coef[m, 1] * xs[None, None, :] + coef[m, 2] * ys[None, :, None]
                 + coef[m, 3] * hc[:, None, None])
    u0 = oracle.interp_wind(uc, xc0, yc0, DXc, DYc, hc, X, Y, Z)
    assert u0.shape == (3,) + xe.shape
    assert xe.min() >= xs[0] and xe.max() <= xs[-1] and he.min() >= hc[0] and he.max() <= hc[-1]
    for m in range(3):
        want = coef[m, 0] + coef[m, 1] * xe + coef[m, 2] * ye + coef[m, 3] * he
        np.testing.assert_allclose(u0[m], want, rtol=0, atol=1e-12 * np.abs(want).max())


def test_interp_clamps_outside_the_coarse_grid():
    """Heights below hc[0] take the hc[0] value; positions beyond the coarse
    grid take the boundary value (constant extension)."""
    X, Y, Z = _hill_mesh()
    xe, ye, he = _centres(X, Y, Z)
    hc = np.array([he.max() + 1.0, he.max() + 2.0])    # every centre is below hc[0]
    uc = np.zeros((3, 2, 2, 2))
    uc[0, 0] = 7.0                                       # level 0: u = 7
    uc[0, 1] = -3.0
    uc[1] = 1.5
    u0 = oracle.interp_wind(uc, 1e6, 1e6, 10.0, 10.0, hc, X, Y, Z)   # grid far away
    np.testing.assert_array_equal(u0[0], 7.0)
    np.testing.assert_array_equal(u0[1], 1.5)
    np.testing.assert_array_equal(u0[2], 0.0)

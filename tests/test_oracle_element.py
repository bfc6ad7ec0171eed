"""Pins of the oracle's element-level arithmetic (Sec. 2)
against closed forms that do not share its code path."""
import json
import os

import numpy as np
import pytest

import oracle
from brute import M2, S2

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))

UNIT = np.array([[a & 1, (a >> 1) & 1, (a >> 2) & 1] for a in range(8)], dtype=float)


def terrain_element(rng, dx=30.0, dy=20.0):
    """Element of a terrain-following grid: rectangular base, bilinear bottom
    and top surfaces (x depends on i only, y on j only)."""
    zb = rng.uniform(0, 10, 4)
    zt = zb + rng.uniform(5, 15, 4)
    xe = np.zeros((8, 3))
    for a in range(8):
        da, db, dc = a & 1, (a >> 1) & 1, (a >> 2) & 1
        xe[a] = [da * dx, db * dy, (zt if dc else zb)[da + 2 * db]]
    vol = dx * dy * np.mean(zt - zb)
    return xe, vol


def random_hex(rng):
    """Randomly perturbed unit cube (positive Jacobian)."""
    return UNIT * rng.uniform(0.5, 2.0, 3) + rng.uniform(-0.12, 0.12, (8, 3))


def test_shape_grad_pins():
    g = GOLD["shape_grad"]
    G = oracle.shape_grad([0, 0, 0])
    s = 2 * UNIT - 1
    np.testing.assert_array_equal(G, g["centre_abs"] * s)
    G = oracle.shape_grad([1, 1, 1])
    np.testing.assert_allclose(G[7], g["corner_111_own"], rtol=0, atol=1e-15)
    rng = np.random.default_rng(0)
    for _ in range(10):
        G = oracle.shape_grad(rng.uniform(-1, 1, 3))
        np.testing.assert_allclose(G.sum(0), 0, atol=1e-15)


def test_unit_cube_stiffness_closed_form():
    g = GOLD["unit_cube_stiffness"]
    K = oracle.element_stiffness(UNIT, [1, 1, 1])
    for a in range(8):
        for b in range(8):
            nd = bin(a ^ b).count("1")
            want = {0: g["diagonal"], 1: g["edge"], 2: g["face"], 3: g["body"]}[nd]
            assert abs(K[a, b] - want) <= 1e-15, (a, b, K[a, b], want)


@pytest.mark.parametrize("h,c", [((1, 1, 1), (1, 1, 1)), ((2.0, 0.5, 3.0), (1, 1, 1)),
                                 ((30.0, 20.0, 7.0), (1.0, 0.25, 0.01)),
                                 ((1.0, 1.0, 1.0), (0.25, 1, 1))])
def test_box_stiffness_kronecker(h, c):
    """Box h1 x h2 x h3 with A^-1 = diag(c): 2-point Gauss is exact, so
    Ke = c1 (h2h3/h1) Mz(x)My(x)Sx + c2 (h1h3/h2) Mz(x)Sy(x)Mx + c3 (h1h2/h3) Sz(x)My(x)Mx
    (local order a = da + 2db + 4dc).  SPEC.md:163 anisotropic example."""
    h1, h2, h3 = h
    xe = UNIT * np.array(h)
    K = oracle.element_stiffness(xe, c)
    k = np.kron
    ref = (c[0] * h2 * h3 / h1 * k(M2, k(M2, S2)) + c[1] * h1 * h3 / h2 * k(M2, k(S2, M2))
           + c[2] * h1 * h2 / h3 * k(S2, k(M2, M2)))
    np.testing.assert_allclose(K, ref, rtol=0, atol=4e-16 * np.abs(ref).max() * 10)


def test_stiffness_invariants_distorted():
    rng = np.random.default_rng(1)
    for _ in range(20):
        xe = random_hex(rng)
        c = rng.uniform(0.01, 1, 3)
        K = oracle.element_stiffness(xe, c)
        assert np.array_equal(K, K.T)                       # exact symmetry
        np.testing.assert_allclose(K.sum(1), 0, atol=1e-14 * np.abs(K).max())
        w = np.linalg.eigvalsh(K)
        assert w[0] > -1e-13 * w[-1]                         # PSD, constant kernel
        assert np.sum(w > 1e-10 * w[-1]) == 7                # rank 7 (2x2x2 Gauss)


def test_linear_energy_exact_on_terrain_elements():
    """For lambda linear (lambda_a = g . x_a), 2x2x2 Gauss integrates exactly on
    trilinear elements: lambda^T Ke lambda = g^T C g vol(e); for a terrain
    column element vol = dx dy mean(dz) (bilinear bottom/top surfaces)."""
    rng = np.random.default_rng(2)
    for _ in range(20):
        xe, vol = terrain_element(rng)
        c = rng.uniform(0.01, 1, 3)
        g = rng.normal(size=3)
        lam = xe @ g
        K = oracle.element_stiffness(xe, c)
        e = lam @ K @ lam
        want = (g * c) @ g * vol
        assert abs(e - want) <= 1e-12 * abs(want)


def test_linear_patch_rows_exact():
    """K lambda_lin row a = int grad N_a . C g; summed over a it is 0 and for
    a box it equals the closed form of the 1-D integrals."""
    rng = np.random.default_rng(3)
    xe = UNIT * np.array([3.0, 2.0, 5.0])
    c = np.array([1.0, 0.5, 0.1])
    g = rng.normal(size=3)
    r = oracle.element_stiffness(xe, c) @ (xe @ g)
    # int_e dN_a/dx_m = s_m * (area of the face orthogonal to m)/4
    s = 2 * UNIT - 1
    area = np.array([2.0 * 5.0, 3.0 * 5.0, 3.0 * 2.0])
    want = (s * area / 4.0) @ (c * g)
    np.testing.assert_allclose(r, want, rtol=0, atol=1e-13)


def test_unit_cube_rhs():
    g = GOLD["unit_cube_rhs"]
    fe = oracle.element_rhs(UNIT, g["u0"])
    for a in range(8):
        want = g["x0_nodes"] if (a & 1) == 0 else g["x1_nodes"]
        assert abs(fe[a] - want) <= 1e-16


def test_box_rhs_closed_form_and_sum():
    rng = np.random.default_rng(4)
    s = 2 * UNIT - 1
    for _ in range(5):
        h = rng.uniform(0.5, 40, 3)
        u = rng.normal(size=3)
        fe = oracle.element_rhs(UNIT * h, u)
        want = -(h.prod() / 4.0) * (s * (u / h)).sum(1)
        np.testing.assert_allclose(fe, want, rtol=1e-14, atol=1e-14 * np.abs(want).max())
    for _ in range(10):
        fe = oracle.element_rhs(random_hex(rng), rng.normal(size=3))
        assert abs(fe.sum()) <= 1e-14 * np.abs(fe).max()


def test_rhs_linear_functional_terrain():
    """One-point rule: fe . lambda_lin = -8 detJ(0) g.u0 and 8 detJ(0) = vol for
    terrain column elements."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        xe, vol = terrain_element(rng)
        g = rng.normal(size=3)
        u = rng.normal(size=3)
        fe = oracle.element_rhs(xe, u)
        want = -vol * (g @ u)
        assert abs(fe @ (xe @ g) - want) <= 1e-12 * (vol * np.abs(g).max() * np.abs(u).max())


def test_centre_gradient_reproduces_linear():
    """Isoparametric elements reproduce linear functions exactly: grad of the
    interpolant of g.x is g at every point, in particular the centre."""
    rng = np.random.default_rng(6)
    for _ in range(20):
        xe = random_hex(rng) if _ % 2 else terrain_element(rng)[0]
        g = rng.normal(size=3)
        np.testing.assert_allclose(oracle.element_grad_centre(xe, xe @ g), g, rtol=0,
                                   atol=1e-12 * np.abs(g).max() * 30)


def test_onepoint_stiffness_rank3_and_agrees_on_linear():
    """C12: K1e has rank 3 and agrees with Ke on linear lambda for box cells."""
    rng = np.random.default_rng(7)
    xe = UNIT * np.array([2.0, 3.0, 0.7])
    c = np.array([1, 1, 0.01])
    K = oracle.element_stiffness(xe, c)
    K1 = oracle.element_stiffness_onepoint(xe, c)
    w = np.linalg.eigvalsh(K1)
    assert np.sum(w > 1e-12 * w[-1]) == 3
    g = rng.normal(size=3)
    np.testing.assert_allclose(K @ (xe @ g), K1 @ (xe @ g), atol=1e-13)


def test_negative_jacobian_detected():
    xe = UNIT.copy()
    xe[[0, 4]] = xe[[4, 0]]
    with pytest.raises(ValueError):
        oracle.element_stiffness(xe, [1, 1, 1])

"""Independent brute-force constructions used to pin the oracle.

Nothing here calls the oracle's arithmetic: these are textbook closed forms
(1-D stiffness/mass Kronecker sums on box grids, fast diagonalisation), dense
linear algebra (numpy/scipy) and the index-space prolongation weights written
out as dense matrices from the paper's definition.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

S2 = np.array([[1.0, -1.0], [-1.0, 1.0]])
M2 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])


def fem1d(h):
    """1-D linear-element stiffness and mass for element lengths h."""
    n = len(h) + 1
    S = np.zeros((n, n))
    M = np.zeros((n, n))
    for e, he in enumerate(h):
        S[e:e + 2, e:e + 2] += S2 / he
        M[e:e + 2, e:e + 2] += M2 * he
    return S, M


def box_stiffness_dense(hx, hy, hz, c):
    """Assembled K of a flat box grid (natural ordering, i fastest):
    K = c1 Mz(x)My(x)Sx + c2 Mz(x)Sy(x)Mx + c3 Sz(x)My(x)Mx."""
    Sx, Mx = fem1d(hx)
    Sy, My = fem1d(hy)
    Sz, Mz = fem1d(hz)
    k = np.kron
    return (c[0] * k(Mz, k(My, Sx)) + c[1] * k(Mz, k(Sy, Mx)) + c[2] * k(Sz, k(My, Mx)))


def free_mask(shape):
    n3, n2, n1 = shape
    m = np.ones(shape, dtype=bool)
    m[-1] = False
    m[:, 0, :] = False
    m[:, -1, :] = False
    m[:, :, 0] = False
    m[:, :, -1] = False
    return m


def _shift_slices(n, d):
    """slices (src, dst) so that dst index t corresponds to src index t + d."""
    if d >= 0:
        return slice(d, n), slice(0, n - d)
    return slice(0, n + d), slice(-d, n)


def neighbour_view(a, dx, dy, dz, fill=0):
    """b[k,j,i] = a[k+dz, j+dy, i+dx] (fill outside the grid)."""
    n3, n2, n1 = a.shape[:3]
    b = np.full_like(a, fill)
    sx, tx = _shift_slices(n1, dx)
    sy, ty = _shift_slices(n2, dy)
    sz, tz = _shift_slices(n3, dz)
    b[tz, ty, tx] = a[sz, sy, sx]
    return b


def free_pair_mask(shape):
    """(n3,n2,n1,27) mask of couplings K[p, o] with both p and p + d_o free."""
    fm = free_mask(shape)
    m = np.zeros(shape + (27,), dtype=bool)
    for o in range(27):
        dx, dy, dz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
        m[..., o] = fm & neighbour_view(fm, dx, dy, dz, False)
    return m


def stencil_asymmetry(K):
    """max |K[p, o] - K[p + d_o, 26 - o]| over in-grid pairs."""
    worst = 0.0
    for o in range(27):
        dx, dy, dz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
        other = neighbour_view(K[..., 26 - o], dx, dy, dz, np.nan)
        d = np.abs(K[..., o] - other)
        worst = max(worst, float(np.nanmax(d)) if np.isfinite(d).any() else 0.0)
    return worst


def fast_diag_solve(hx, hy, hz, c, f):
    """lambda* = K_FF^{-1} f_F on a flat box by fast diagonalisation: 1-D
    generalised eigenproblems S v = mu M v restricted to the free index set of
    each direction (Dirichlet at both x/y ends and at the top, natural at the
    bottom).  f: (n3, n2, n1) array; returns (n3, n2, n1) with zeros on D."""
    Sx, Mx = fem1d(hx)
    Sy, My = fem1d(hy)
    Sz, Mz = fem1d(hz)
    fx = slice(1, len(hx))          # interior x nodes
    fy = slice(1, len(hy))
    fz = slice(0, len(hz))          # bottom free, top Dirichlet
    mux, Vx = sla.eigh(Sx[fx, fx], Mx[fx, fx])
    muy, Vy = sla.eigh(Sy[fy, fy], My[fy, fy])
    muz, Vz = sla.eigh(Sz[fz, fz], Mz[fz, fz])
    F = f[fz, fy, fx]
    # V^T f
    G = np.einsum("ai,bj,ck,cba->kji", Vx, Vy, Vz, F, optimize=True)
    lam = (c[0] * mux[None, None, :] + c[1] * muy[None, :, None] + c[2] * muz[:, None, None])
    G = G / lam
    X = np.einsum("ai,bj,ck,kji->cba", Vx, Vy, Vz, G, optimize=True)
    out = np.zeros_like(f)
    out[fz, fy, fx] = X
    return out


def prolong1d(n, kept):
    """Dense 1-D index-space trilinear prolongation: coarse node c
    at fine index kept[c]; a fine node between two kept nodes two apart gets
    1/2, 1/2."""
    m = len(kept)
    P = np.zeros((n, m))
    for c, t in enumerate(kept):
        P[t, c] = 1.0
    for c in range(m - 1):
        a, b = kept[c], kept[c + 1]
        assert b - a in (1, 2)
        if b - a == 2:
            P[a + 1, c] = 0.5
            P[a + 1, c + 1] = 0.5
    return P


def horizontal_kept(n):
    k = list(range(0, n, 2))
    if k[-1] != n - 1:
        k.append(n - 1)
    return k


def prolong_dense(shape, horizontal, kept_z):
    n3, n2, n1 = shape
    kx = horizontal_kept(n1) if horizontal else list(range(n1))
    ky = horizontal_kept(n2) if horizontal else list(range(n2))
    P = np.kron(prolong1d(n3, kept_z), np.kron(prolong1d(n2, ky), prolong1d(n1, kx)))
    return P, (len(kept_z), len(ky), len(kx))


def gs_order(shape):
    """Free nodes in the smoother's order: colour (0,0),(1,0),(0,1),(1,1) of
    (i mod 2, j mod 2), then column (j, i), then k bottom-up."""
    n3, n2, n1 = shape
    colours = [(0, 0), (1, 0), (0, 1), (1, 1)]
    order = []
    for (ci, cj) in colours:
        for j in range(1, n2 - 1):
            if j % 2 != cj:
                continue
            for i in range(1, n1 - 1):
                if i % 2 != ci:
                    continue
                for k in range(0, n3 - 1):
                    order.append((k * n2 + j) * n1 + i)
    return np.array(order)


def gs_dense(A, f, x, order):
    """One Gauss-Seidel sweep in the given order as a dense triangular solve:
    x_new = (D + L)^{-1} (f - U x_old) on the permuted free block."""
    Ap = A[np.ix_(order, order)]
    L = np.tril(Ap)
    U = np.triu(Ap, 1)
    xo = x.ravel()[order]
    xn = sla.solve_triangular(L, f.ravel()[order] - U @ xo, lower=True)
    out = x.ravel().copy()
    out[order] = xn
    return out.reshape(x.shape)


def line_dense(A, f, x, shape):
    """One block Gauss-Seidel sweep whose blocks are the free vertical columns,
    in the smoother's colour order (0,0),(1,0),(0,1),(1,1), each block solved
    exactly with numpy (dense) given the latest values of all other nodes:
    x_c <- A_cc^{-1} (f_c - sum_{q not in c} A_cq x_q).  Independent of the
    oracle's Thomas recurrences."""
    n3, n2, n1 = shape
    m = free_mask(shape).ravel()
    xv = x.ravel().copy()
    fv = f.ravel()
    for (ci, cj) in [(0, 0), (1, 0), (0, 1), (1, 1)]:
        for j in range(1, n2 - 1):
            if j % 2 != cj:
                continue
            for i in range(1, n1 - 1):
                if i % 2 != ci:
                    continue
                idx = np.array([(k * n2 + j) * n1 + i for k in range(n3 - 1)])
                rest = m.copy()
                rest[idx] = False
                r = fv[idx] - A[np.ix_(idx, np.flatnonzero(rest))] @ xv[rest]
                xv[idx] = np.linalg.solve(A[np.ix_(idx, idx)], r)
    return xv.reshape(shape)

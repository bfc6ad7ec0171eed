"""Parity at BASELINE.json's full sizes (Medium 1000x1000x15, Paper-scale
3000x3000x15), in the launch configuration bench.py times (default options,
CUDA graph), on sampled outputs the oracle computes one by one from its
element routines, plus properties that hold at any size:
  * stencil rows (27 couplings) at sampled nodes: <= 1e-12 relative;
  * RHS at sampled nodes, recovered wind at sampled elements: <= 1e-12;
  * K lambda of the converged GPU solution at sampled nodes (oracle element
    matrices times the GPU lambda) vs the GPU apply there: <= 1e-12 of
    sum |K_o lambda_o|; the GPU's relative residual <= 1e-8 and the sampled
    pointwise residual small against max|f|;
  * lambda = 0 on the Dirichlet set, exactly.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
NS = 160   # sampled nodes / elements per check


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _elem_xe(X, Y, Z, i, j, k):
    xe = np.zeros((8, 3))
    for a in range(8):
        ii, jj, kk = i + (a & 1), j + ((a >> 1) & 1), k + ((a >> 2) & 1)
        xe[a] = [X[kk, jj, ii], Y[kk, jj, ii], Z[kk, jj, ii]]
    return xe


def _node_row27(X, Y, Z, a, i, j, k):
    """27 couplings of node (i,j,k) summed over its elements (oracle element matrices)."""
    n3, n2, n1 = X.shape
    c = 1.0 / np.asarray(a, dtype=float) ** 2
    row = np.zeros(27)
    for ek in (k - 1, k):
        for ej in (j - 1, j):
            for ei in (i - 1, i):
                if not (0 <= ei < n1 - 1 and 0 <= ej < n2 - 1 and 0 <= ek < n3 - 1):
                    continue
                Ke = oracle.element_stiffness(_elem_xe(X, Y, Z, ei, ej, ek), c)
                la = (i - ei) + 2 * (j - ej) + 4 * (k - ek)
                for b in range(8):
                    dx = (ei + (b & 1)) - i
                    dy = (ej + ((b >> 1) & 1)) - j
                    dz = (ek + ((b >> 2) & 1)) - k
                    row[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] += Ke[la, b]
    return row


def _node_rhs(X, Y, Z, U, i, j, k):
    """f at node (i,j,k): sum of the oracle element RHS of its elements; U is
    the (3, nz, ny, nx) element array on the device (read per element)."""
    n3, n2, n1 = X.shape
    s = 0.0
    for ek in (k - 1, k):
        for ej in (j - 1, j):
            for ei in (i - 1, i):
                if not (0 <= ei < n1 - 1 and 0 <= ej < n2 - 1 and 0 <= ek < n3 - 1):
                    continue
                ue = U[:, ek, ej, ei].cpu().numpy()
                fe = oracle.element_rhs(_elem_xe(X, Y, Z, ei, ej, ek), ue)
                s += fe[(i - ei) + 2 * (j - ej) + 4 * (k - ek)]
    return s


@pytest.fixture(scope="module", params=["medium", "paper"])
def big(request, wd):
    p = synth.make(request.param, device=DEV)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)              # bench.py's default options
    f = wd.wd_rhs(ctx, p.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-8)
    rng = np.random.default_rng(17)
    n1, n2, n3 = p.dims
    nodes = np.stack([rng.integers(1, n1 - 1, NS), rng.integers(1, n2 - 1, NS),
                      rng.integers(0, n3 - 1, NS)], 1)
    nodes[:8, 2] = 0                                       # include the terrain (Gamma) layer
    elems = np.stack([rng.integers(0, n1 - 1, NS), rng.integers(0, n2 - 1, NS),
                      rng.integers(0, n3 - 1, NS)], 1)
    # host copies of the neighbourhoods only
    Xh, Yh, Zh = (t.cpu().numpy() for t in (p.X, p.Y, p.Z))
    yield dict(p=p, ctx=ctx, f=f, lam=lam, rep=rep, nodes=nodes, elems=elems, XYZ=(Xh, Yh, Zh))
    ctx.close()


def test_fullsize_stencil_rows(big, wd):
    ctx, p = big["ctx"], big["p"]
    X, Y, Z = big["XYZ"]
    K = wd.wd_get_stencil(ctx, 0)                          # (n3, n2, n1, 27) on the device
    idx = torch.as_tensor(big["nodes"], device=DEV)
    got = K[idx[:, 2], idx[:, 1], idx[:, 0]].cpu().numpy()
    del K
    torch.cuda.empty_cache()
    for s, (i, j, k) in enumerate(big["nodes"]):
        want = _node_row27(X, Y, Z, p.a, i, j, k)
        assert np.abs(got[s] - want).max() <= 1e-12 * np.abs(want).max(), (i, j, k)


def test_fullsize_rhs_and_recovery(big, wd):
    ctx, p = big["ctx"], big["p"]
    X, Y, Z = big["XYZ"]
    U = p.u0
    f = big["f"]
    fmax = float(f.abs().max())
    for (i, j, k) in big["nodes"][:60]:
        want = _node_rhs(X, Y, Z, U, i, j, k)
        assert abs(float(f[k, j, i]) - want) <= 1e-12 * fmax, (i, j, k)
    lam = big["lam"]
    u = wd.wd_recover_wind(ctx, lam, U)
    c = 1.0 / np.asarray(p.a) ** 2
    lh = lam
    for (i, j, k) in big["elems"]:
        xe = _elem_xe(X, Y, Z, i, j, k)
        la = np.array([float(lh[k + ((a >> 2) & 1), j + ((a >> 1) & 1), i + (a & 1)])
                       for a in range(8)])
        g = oracle.element_grad_centre(xe, la)
        want = U[:, k, j, i].cpu().numpy() + c * g
        gotv = u[:, k, j, i].cpu().numpy()
        assert np.abs(gotv - want).max() <= 1e-12 * np.abs(want).max()


def test_fullsize_solution_residual(big, wd):
    """The converged lambda satisfies the discrete equations (Eq. (5)) at the
    sampled nodes: oracle element matrices x GPU lambda - f."""
    ctx, p = big["ctx"], big["p"]
    X, Y, Z = big["XYZ"]
    lam, f, rep = big["lam"], big["f"], big["rep"]
    assert rep["converged"] and rep["rel_res_final"] <= 1e-8
    Klam = wd.wd_apply(ctx, 0, lam)
    fmax = float(f.abs().max())
    fnorm = float(torch.linalg.vector_norm(f))            # |r_i| <= ||r||_2 = rel_res ||f||_2
    for (i, j, k) in big["nodes"][:80]:
        row = _node_row27(X, Y, Z, p.a, i, j, k)
        nb = np.zeros(27)
        for o in range(27):
            dx, dy, dz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
            kk = k + dz
            if 0 <= kk < p.dims[2]:
                nb[o] = float(lam[kk, j + dy, i + dx])
        want = row @ nb
        # rounding bound of a 27-term dot product: a few ulps of sum |row_o nb_o|
        assert abs(float(Klam[k, j, i]) - want) <= 1e-12 * float(np.abs(row * nb).sum()), (i, j, k)
        # and the solution satisfies the equation there to the solve's tolerance
        assert abs(want - float(f[k, j, i])) <= 1.01 * rep["rel_res_final"] * fnorm + 1e-12 * fmax
    # exact zeros on the Dirichlet set
    assert not lam[-1].any() and not lam[:, 0].any() and not lam[:, -1].any()
    assert not lam[:, :, 0].any() and not lam[:, :, -1].any()


def test_fullsize_sweep_gs_equations(big, wd):
    """One fused smoother sweep at full size, checked against the
    oracle's element matrices at sampled nodes of the LAST colour (i, j odd):
    when they are updated every neighbour is final except the one above in the
    same column (bottom-up: still the input value), so
    K_pp x_p = f_p - sum_{q != p} K_pq x_q  with x_q the output, and the input
    for q = p + (0,0,1), holds to rounding; and the fused sweep equals the four
    colour-phase launches bit for bit."""
    ctx, p = big["ctx"], big["p"]
    X, Y, Z = big["XYZ"]
    n1, n2, n3 = p.dims
    g = torch.Generator(device=DEV).manual_seed(5)
    x0 = torch.rand((n3, n2, n1), dtype=torch.float64, device=DEV, generator=g) * 2 - 1
    f = big["f"]
    x1 = wd.wd_smooth(ctx, 0, x0.clone(), f, sweeps=1)
    rng = np.random.default_rng(23)
    pts = np.stack([2 * rng.integers(0, (n1 - 2) // 2, 60) + 1, 2 * rng.integers(0, (n2 - 2) // 2, 60) + 1,
                    rng.integers(0, n3 - 1, 60)], 1)
    for (i, j, k) in pts:
        row = _node_row27(X, Y, Z, p.a, i, j, k)
        nb = np.zeros(27)
        for o in range(27):
            dx, dy, dz = o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1
            kk = k + dz
            if 0 <= kk < n3:
                nb[o] = float(x1[kk, j + dy, i + dx])
        # the node above: its input value (0 on the Dirichlet top plane)
        nb[22] = float(x0[k + 1, j, i]) if k + 1 < n3 - 1 else 0.0
        r = float(f[k, j, i]) - row @ nb
        assert abs(r) <= 1e-12 * (float(np.abs(row * nb).sum()) + abs(float(f[k, j, i]))), (i, j, k)
    # the same sweep as four colour-phase launches (a second context, phased)
    opt = wd.default_options(smoother="phased")
    cph = wd.wd_assemble(p.X, p.Y, p.Z, p.a, opt)
    x2 = wd.wd_smooth(cph, 0, x0.clone(), f, sweeps=1)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)
    cph.close()

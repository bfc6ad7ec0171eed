"""Degenerate and extreme grid shapes against the oracle: a single free
column, one element layer, rows or columns of width 2, a 200-layer column
(the line smoother's shared-memory Thomas path holds <= 32 planes, so this
takes its HBM scratch path), and grids whose hierarchy coarsens in one
direction only.  For each: the hierarchy equals the oracle's, the stencil /
RHS / operator / recovery <= 1e-12 relative max, and the solve to 1e-10 gives
lambda <= 1e-8 relative l2 and cycles +- 1 (north_star tolerances).
(Dirichlet set), P:107-114 (assembly, RHS, recovery), Eq. (7) (multigrid).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import free_mask

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _noisy(p, seed):
    g = torch.Generator().manual_seed(seed)
    u0 = p.u0 + 0.5 * torch.randn(p.u0.shape, generator=g, dtype=torch.float64)
    return synth.Problem(p.name, p.nx, p.ny, p.nz, p.X, p.Y, p.Z, u0, p.a, p.meta)


SHAPES = {
    # (nx, ny, nz), hill height, a
    "one_column": ((2, 2, 1), 10.0, (1, 1, 1)),
    "one_column_deep": ((2, 2, 9), 10.0, (1, 1, 10)),
    "one_layer": ((23, 17, 1), 60.0, (1, 1, 1)),
    "thin_x": ((2, 31, 6), 60.0, (1, 1, 3)),
    "thin_y": ((29, 2, 6), 60.0, (1, 1, 3)),
    "three_wide": ((3, 3, 4), 30.0, (1, 2, 5)),
    "tall_200": ((6, 5, 200), 80.0, (1, 1, 10)),
    "strip": ((97, 4, 5), 90.0, (1, 1, 10)),
}


def _problem(name):
    (nx, ny, nz), h, a = SHAPES[name]
    dz0, r = (2.0, 1.01) if nz > 100 else (6.0, 1.2)
    p = synth.hill(nx=nx, ny=ny, nz=nz, dx=25.0, height=h, sigma=max(nx, ny) * 8.0,
                   dz0=dz0, r=r, a=a, u0=(4.0, -1.5, 0.3))
    return _noisy(p, 7)


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _n(t):
    return t.detach().cpu().numpy()


def _rel_max(a, b):
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


@pytest.mark.parametrize("smoother", ["fused", "line"])
@pytest.mark.parametrize("name", list(SHAPES))
def test_edge_shapes_parity(wd, name, smoother):
    p = _problem(name)
    X, Y, Z, u0 = p.numpy()
    cmax = 6
    opt = wd.default_options(coarsest_max_free=cmax, smoother=smoother)
    g = p.to(DEV)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=cmax,
                   smoother="gs" if smoother == "fused" else "line")
    try:
        assert [tuple(ctx.level_dims(l)) for l in range(ctx.num_levels())] == \
            [tuple(d) for d in mg.dims]
        for l in range(mg.nlev):
            x = np.random.default_rng(l).uniform(-1, 1, mg.shape(l)) * free_mask(mg.shape(l))
            y = _n(wd.wd_apply(ctx, l, torch.as_tensor(x, device=DEV)))
            assert _rel_max(y, mg.apply(l, x)) <= 1e-12, l
        f = wd.wd_rhs(ctx, g.u0)
        fo = oracle.rhs(X, Y, Z, u0)
        assert _rel_max(_n(f), fo) <= 1e-12
        lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
        lo, ro = mg.solve(fo, tol=1e-10)
        assert np.linalg.norm(_n(lam) - lo) <= 1e-8 * max(np.linalg.norm(lo), 1e-300)
        assert abs(rep["cycles"] - ro["cycles"]) <= 1, (rep["cycles"], ro["cycles"])
        u = _n(wd.wd_recover_wind(ctx, lam, g.u0))
        uo = oracle.recover(X, Y, Z, p.a, lo, u0)
        assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    finally:
        ctx.close()


def test_edge_shape_limits(wd):
    """The smallest grid (3 x 3 x 2 nodes) is accepted; n1 or n2 < 3, n3 < 2
    and n3 - 1 >= 512 layers are rejected with WD_E_INVAL before any work."""
    for dims, ok in [((3, 3, 2), True), ((2, 3, 2), False), ((3, 2, 2), False),
                     ((3, 3, 1), False), ((3, 3, 513), False)]:
        n1, n2, n3 = dims
        p = synth.box(n1 - 1, n2 - 1, max(n3 - 1, 1), dx=10.0, dy=10.0, dz=1.0, device=DEV)
        X, Y, Z = (t[:n3].contiguous() for t in (p.X, p.Y, p.Z))
        if n3 > p.X.shape[0]:
            X, Y, Z = (t[:1].expand(n3, n2, n1).contiguous() for t in (p.X, p.Y, p.Z))
            Z = Z + torch.arange(n3, dtype=torch.float64, device=DEV).view(-1, 1, 1)
        if ok:
            wd.wd_assemble(X, Y, Z, (1.0, 1.0, 1.0)).close()
        else:
            with pytest.raises(wd.WDError) as e:
                wd.wd_assemble(X, Y, Z, (1.0, 1.0, 1.0))
            assert e.value.code == wd.WD_E_INVAL

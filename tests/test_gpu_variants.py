"""GPU-vs-oracle parity for the paper's variants and the solve loop's guards:

  * coarsest level by "more iterations" instead of the direct solve
    (reading C8: 50 GS sweeps from zero when the planner stops above
    coarsest_max_free; forced here with coarsest_max_free = 0), alone and with
    the base method's full 2x2x2 coarsening (WD_RULE_FULL);
  * the planner's inputs (reading C2) on hand-built grids whose
    minimum-terrain column (with ties) decides the hierarchy;
  * WD_E_NONFINITE (a NaN in f) and WD_E_DIVERGED (the S:355 rule, provoked by
    an over-weighted coarse-grid correction through the test-only knob
    WD_TEST_CORRECTION_WEIGHT).
Tolerances as tests/test_gpu_parity.py: one V-cycle <= 1e-10 relative max
(both sides run the same GS sweeps at the coarsest level, so this is rounding
only), lambda after both reach 1e-10 <= 1e-8 relative l2, cycles +-1, rate
within 10 %.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from test_oracle_planner_inputs import _grid

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _n(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


GRIDS = {
    "tiny": lambda: synth.tiny(),
    "ragged": lambda: synth.hill(nx=37, ny=22, nz=5, dx=40.0, height=120.0, sigma=300.0,
                                 dz0=8.0, r=1.3, a=(1, 1, 3)),
}


@pytest.mark.parametrize("rule", ["coupling_cur", "full"])
@pytest.mark.parametrize("grid", list(GRIDS))
def test_coarse_iterative_parity(wd, grid, rule):
    p = GRIDS[grid]()
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    opt = wd.default_options(coarsest_max_free=0, coarsen_rule=rule, max_cycles=200)
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, opt)
    mg = oracle.MG(X, Y, Z, p.a, rule=rule, coarsest_max_free=0)
    assert not mg.coarse_direct
    assert [ctx.level_dims(l) for l in range(ctx.num_levels())] == mg.dims
    f_o = oracle.rhs(X, Y, Z, u0)
    f = wd.wd_rhs(ctx, g.u0)
    # one V-cycle from a random start
    lam0 = synth.random_lambda(p, 3).numpy()
    v = torch.as_tensor(lam0, device=DEV).clone()
    wd.wd_vcycle(ctx, v, f, want_residual=False)
    vo = mg.vcycle(lam0, f_o)
    assert np.abs(_n(v) - vo).max() <= 1e-10 * np.abs(vo).max()
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10, raise_on_noconv=False)
    assert rep["coarse_direct"] is False
    lo, ro = mg.solve(f_o, tol=1e-10, max_cycles=200)
    assert rep["status"] == ro["status"] == 0
    assert abs(rep["cycles"] - ro["cycles"]) <= 1
    assert abs(rep["rate"] - ro["rate"]) <= 0.1 * ro["rate"]
    assert np.linalg.norm(_n(lam) - lo) <= 1e-8 * np.linalg.norm(lo)
    ctx.close()


def _tie_grid():
    # three columns tie at the minimum terrain height (linear indices 11, 20,
    # 24); the first one has thin layers (no horizontal coarsening, layers
    # merged), the others and the rest thick layers (horizontal coarsening)
    n1, n2 = 6, 5
    zs = np.full((n2, n1), 50.0)
    for (i, j) in [(5, 1), (2, 3), (0, 4)]:
        zs[j, i] = -4.0

    def layers(i, j):
        if (i, j) == (5, 1):
            return [2.0, 2.5, 3.0, 3.5]
        return [(k + 1) * (40.0 + i + j) for k in range(4)]
    return _grid(n1, n2, 25.0, 25.0, zs, layers)


def test_planner_inputs_gpu(wd):
    X, Y, Z = _tie_grid()
    a = (1.0, 1.0, 1.0)
    h1, h3 = oracle.planner_inputs(X, Y, Z)
    np.testing.assert_array_equal(h3, [2.0, 2.5, 3.0, 3.5])   # the first tie's column
    want = oracle.plan_level(h1, h3, a, n1=6, n2=5)
    assert not want["horizontal"] and want["kept"] == [0, 2, 4]
    mg = oracle.MG(X, Y, Z, a, coarsest_max_free=1)
    assert mg.plans[0] == {"horizontal": want["horizontal"], "kept": want["kept"]}
    t = [torch.as_tensor(v, device=DEV) for v in (X, Y, Z)]
    ctx = wd.wd_assemble(*t, a, wd.default_options(coarsest_max_free=1))
    assert [ctx.level_dims(l) for l in range(ctx.num_levels())] == mg.dims
    for l in range(mg.nlev - 1):
        assert ctx.level_plan(l) == mg.plans[l]
    ctx.close()


def test_nonfinite_residual(wd):
    p = synth.tiny().to(DEV)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60))
    f = wd.wd_rhs(ctx, p.u0)
    f[3, 5, 7] = float("nan")
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-8, raise_on_noconv=False)
    assert rep["status"] == wd.WD_E_NONFINITE
    with pytest.raises(wd.WDError) as e:
        wd.wd_solve(ctx, f, rel_tol=1e-8)
    assert e.value.code == wd.WD_E_NONFINITE
    # the context is still usable: a finite f solves normally afterwards
    f = wd.wd_rhs(ctx, p.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
    assert rep["converged"]
    ctx.close()


def test_diverged_guard(wd):
    """rel_c > 10 rel_{c-3} stops the solve with WD_E_DIVERGED.  A
    coarse-grid correction weighted by 4 (lam += 4 P lam_c) over-corrects the
    smooth error by a factor -3 per cycle, which the smoother does not damp."""
    p = synth.tiny().to(DEV)
    os.environ["WD_TEST_CORRECTION_WEIGHT"] = "4"
    try:
        ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60))
    finally:
        del os.environ["WD_TEST_CORRECTION_WEIGHT"]
    f = wd.wd_rhs(ctx, p.u0)
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10, raise_on_noconv=False)
    assert rep["status"] == wd.WD_E_DIVERGED, rep
    c = rep["cycles"]
    assert c >= 3 and rep["hist"][c] > 10 * rep["hist"][c - 3]
    ctx.close()
    # the weight is per context: a new context solves normally
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60))
    lam, rep = wd.wd_solve(ctx, wd.wd_rhs(ctx, p.u0), rel_tol=1e-10)
    assert rep["converged"]
    ctx.close()


@pytest.mark.parametrize("line_from", [1, 2])
@pytest.mark.parametrize("grid", ["small", "ragged"])
def test_per_level_smoother_parity(wd, grid, line_from):
    """Per-level smoother (SURVEY 8(f) f1 "per-level decisions"): the fused
    point GS on the levels below `line_from`, vertical line
    relaxation (reading C19) from it on -- GPU and oracle with the same
    choice: hierarchy, one V-cycle <= 1e-10, the solve to 1e-10 (cycles +-1,
    rate within 10 %, lambda <= 1e-8), bitwise-equal re-solve."""
    p = synth.small() if grid == "small" else GRIDS["ragged"]()
    X, Y, Z, u0 = p.numpy()
    g = p.to(DEV)
    cmax = 4096 if grid == "small" else 60
    ctx = wd.wd_assemble(g.X, g.Y, g.Z, p.a, wd.default_options(coarsest_max_free=cmax,
                                                                 line_from_level=line_from))
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=cmax, line_from_level=line_from)
    assert [ctx.level_dims(l) for l in range(ctx.num_levels())] == mg.dims
    f_o = oracle.rhs(X, Y, Z, u0)
    f = wd.wd_rhs(ctx, g.u0)
    lam0 = synth.random_lambda(p, 4).numpy()
    v = torch.as_tensor(lam0, device=DEV).clone()
    wd.wd_vcycle(ctx, v, f, want_residual=False)
    vo = mg.vcycle(lam0, f_o)
    assert np.abs(_n(v) - vo).max() <= 1e-10 * np.abs(vo).max()
    lam, rep = wd.wd_solve(ctx, f, rel_tol=1e-10)
    lo, ro = mg.solve(f_o, tol=1e-10, max_cycles=100)
    assert ro["status"] == 0 and abs(rep["cycles"] - ro["cycles"]) <= 1
    assert abs(rep["rate"] - ro["rate"]) <= 0.1 * ro["rate"]
    assert np.linalg.norm(_n(lam) - lo) <= 1e-8 * np.linalg.norm(lo)
    lam2, _ = wd.wd_solve(ctx, f, rel_tol=1e-10)
    assert torch.equal(lam, lam2)
    ctx.close()

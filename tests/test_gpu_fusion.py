"""The prolongation (Eq. (7) "u <- u + P u_c") folded into the
first post-smoothing sweep (k_gs_fused2.cu PRO variant, env WD_FUSE_PROLONG=1)
against the separate pass (the default): every V-cycle iterate, the whole
solve and the single-transition entry point bitwise equal, on grids whose
transitions have an identity z map (horizontal coarsening only) mixed with
ones that merge layers, with ragged tails.

The knobs are read at wd_assemble and kept per context.  The oracle parity of
the default path is covered by tests/test_gpu_parity.py; bitwise equality
carries it over to the alternatives."""
import os

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")

GRIDS = {
    "small": lambda: synth.small(device=DEV),
    "ragged": lambda: synth.hill(nx=37, ny=22, nz=5, dx=40.0, height=120.0, sigma=300.0,
                                 dz0=8.0, r=1.3, a=(1, 1, 3), device=DEV),
    "crop": lambda: synth.crop(synth.hill(nx=300, ny=200, nz=12, dx=30.0, height=250.0,
                                          sigma=900.0, dz0=8.0, r=1.2, a=(1, 1, 10)),
                               0, 0, 300, 200).to(DEV),
}


@pytest.fixture(scope="module")
def wd():
    import paper_2101_08453_b200 as m
    return m


def _ctx(wd, p, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


VARIANTS = {
    "fused_prolong": ({"WD_FUSE_PROLONG": "1"}, {"WD_FUSE_PROLONG": "0"}),
}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("grid", list(GRIDS))
def test_prolongation_schedules_bitwise(wd, grid, variant):
    p = GRIDS[grid]()
    ea, eb = VARIANTS[variant]
    a = _ctx(wd, p, ea)
    b = _ctx(wd, p, eb)
    try:
        plans = [a.level_plan(l) for l in range(a.num_levels() - 1)]
        assert any(pl["horizontal"] for pl in plans)
        f = wd.wd_rhs(a, p.u0)
        x = synth.random_lambda(p, 3)
        xa, xb = x.clone(), x.clone()
        for _ in range(3):
            wd.wd_vcycle(a, xa, f, want_residual=False)
            wd.wd_vcycle(b, xb, f, want_residual=False)
            torch.cuda.synchronize()
            assert torch.equal(xa, xb)
        la, ra = wd.wd_solve(a, f, rel_tol=1e-10)
        lb, rb = wd.wd_solve(b, f, rel_tol=1e-10)
        assert torch.equal(la, lb) and ra["cycles"] == rb["cycles"]
        assert ra["hist"] == rb["hist"]
        # the single-transition entry point too
        if a.num_levels() > 1:
            n1, n2, n3 = a.level_dims(1)
            xc = torch.randn(n3, n2, n1, dtype=torch.float64, device=DEV)
            ya = wd.wd_prolong(a, 0, xc, x.clone())
            yb = wd.wd_prolong(b, 0, xc, x.clone())
            assert torch.equal(ya, yb)
    finally:
        a.close()
        b.close()


def test_knobs_are_per_context(wd):
    """Two contexts assembled under different knob settings keep their own
    (the V-cycle graphs are captured at the first cycle, after both exist)."""
    p = GRIDS["small"]()
    a = _ctx(wd, p, {"WD_TEST_GS_GRID": "1"})
    b = _ctx(wd, p, {"WD_TEST_GS_GRID": "0"})
    try:
        f = wd.wd_rhs(a, p.u0)
        ta = wd.wd_bench_kernel(a, "gs_sweep", 0, 3)
        tb = wd.wd_bench_kernel(b, "gs_sweep", 0, 3)
        assert ta > 2 * tb   # one persistent CTA against the full grid
        la, _ = wd.wd_solve(a, f, rel_tol=1e-9)
        lb, _ = wd.wd_solve(b, f, rel_tol=1e-9)
        assert torch.equal(la, lb)
    finally:
        a.close()
        b.close()

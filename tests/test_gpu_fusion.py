"""The prolongation folded into the first post-smoothing sweep (k_gs_fused2.cu
PRO variant, env WD_FUSE_PROLONG=1; Eq. (7) "u <- u + P u_c")
against the separate prolongation pass (the default): every V-cycle iterate
and the whole solve bitwise equal, on grids whose transitions fold
(horizontal, identity z) and mix with ones that do not (vertical merging),
with ragged tails.  The oracle parity of the default path is covered by
tests/test_gpu_parity.py; bitwise equality carries it over to the folded one."""
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


def _ctx(wd, p, fuse):
    old = os.environ.get("WD_FUSE_PROLONG")
    os.environ["WD_FUSE_PROLONG"] = "1" if fuse else "0"
    try:
        return wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(coarsest_max_free=60))
    finally:
        if old is None:
            os.environ.pop("WD_FUSE_PROLONG", None)
        else:
            os.environ["WD_FUSE_PROLONG"] = old


@pytest.mark.parametrize("grid", list(GRIDS))
def test_fused_prolongation_bitwise(wd, grid):
    p = GRIDS[grid]()
    try:
        a = _ctx(wd, p, True)
        b = _ctx(wd, p, False)
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
        a.close()
        b.close()
    finally:
        _ctx(wd, p, False).close()   # the knob is read at assembly: back to the default

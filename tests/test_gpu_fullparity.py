"""Whole-solve parity on Medium (BASELINE configs[2], 1000x1000x15, 16 M
nodes): the GPU path in bench.py's launch configuration against the oracle's
own multigrid solve (tests/parity_full.py).  north_star bars: RHS <= 1e-12
relative max; one V-cycle from zero <= 1e-10 relative max (the coarsest
solves differ: Cholesky in the oracle, a Gauss-Jordan inverse on the GPU,
reading C8, so the V-cycle agrees to O(cond * eps) rather than 1e-12);
lambda and the recovered wind after both reach 1e-10 <= 1e-8 relative l2;
cycles +-1; convergence factor within 10 %; identical hierarchy."""
import pytest
import torch

from parity_full import TOL_F, TOL_LAM, TOL_RATE, solve_parity

pytestmark = pytest.mark.gpu


def test_medium_solve_parity():
    import paper_2101_08453_b200 as wd
    r = solve_parity("medium", wd, torch.device("cuda:0"), tol=1e-10)
    c = r["compare"]
    assert c["levels_equal"]
    assert c["rhs_rel_max"] <= TOL_F
    assert c["vcycle1_rel_max"] <= 1e-10
    assert c["lam_rel_l2"] <= TOL_LAM and c["u_rel_l2"] <= TOL_LAM
    assert abs(c["cycles_diff"]) <= 1
    assert c["rate_rel_diff"] <= TOL_RATE
    assert r["oracle"]["status"] == 0
    assert r["gpu"]["cycles_to_1e8"] is not None

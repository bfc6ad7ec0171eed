"""wd_solve's cycle loop on the device (wd_options.device_loop = 1: one CUDA
graph whose conditional WHILE node repeats the V-cycle while a kernel's
convergence test says so) against the host-driven loop (device_loop = 0, the
default): the same iterate, residual history, cycle count, status
and rate bit for bit, for the zero start, a warm start, the cycle cap
(WD_E_NOCONV), a NaN in f (WD_E_NONFINITE) and an over-weighted correction
(WD_E_DIVERGED; S:195-203, S:351-359 stopping rules, reading C9 "cycle, then
test").  The host loop's own parity with the oracle is tests/test_gpu_parity.py.
"""
import os

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")

GRIDS = {
    "tiny": lambda: synth.tiny(device=DEV),
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


def _pair(wd, p, env=None, **kw):
    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        a = wd.wd_assemble(p.X, p.Y, p.Z, p.a,
                           wd.default_options(coarsest_max_free=60, device_loop=1, **kw))
        b = wd.wd_assemble(p.X, p.Y, p.Z, p.a,
                           wd.default_options(coarsest_max_free=60, device_loop=0, **kw))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return a, b


def _same(wd, a, b, f, lam0=None, tol=1e-10):
    n0 = wd.wd_launch_count()
    la, ra = wd.wd_solve(a, f, lam0=lam0, rel_tol=tol, raise_on_noconv=False)
    torch.cuda.synchronize()
    n1 = wd.wd_launch_count()
    lb, rb = wd.wd_solve(b, f, lam0=lam0, rel_tol=tol, raise_on_noconv=False)
    torch.cuda.synchronize()
    n2 = wd.wd_launch_count()
    assert ra["status"] == rb["status"]
    assert ra["cycles"] == rb["cycles"]
    c = ra["cycles"]
    assert ra["hist"][: c + 1] == rb["hist"][: c + 1] or (
        ra["status"] == wd.WD_E_NONFINITE)
    for k in ("rel_res0", "rel_res_final", "rate"):
        if ra["status"] != wd.WD_E_NONFINITE:
            assert ra[k] == rb[k], k
    assert torch.equal(la, lb) or ra["status"] == wd.WD_E_NONFINITE
    # the same bodies ran: the device loop adds its test kernel per test
    # (c + 1) and its post kernel per cycle
    assert (n1 - n0) - (n2 - n1) == 2 * c + 1, (n1 - n0, n2 - n1, c)
    return ra


@pytest.mark.parametrize("grid", list(GRIDS))
def test_device_loop_zero_and_warm_start(wd, grid):
    p = GRIDS[grid]()
    a, b = _pair(wd, p)
    try:
        f = wd.wd_rhs(a, p.u0)
        r = _same(wd, a, b, f)
        assert r["status"] == wd.WD_OK and r["cycles"] >= 2
        # warm start from a perturbed solution (the residual of lam0 comes from
        # the first sweep's residual variant)
        lam, _ = wd.wd_solve(b, f, rel_tol=1e-6)
        lam0 = lam + 1e-3 * synth.random_lambda(p, 5)
        _same(wd, a, b, f, lam0=lam0, tol=1e-9)
        # repeated solves reuse the graph
        _same(wd, a, b, f, tol=1e-7)
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("cap", [0, 1, 3])
def test_device_loop_cycle_cap(wd, cap):
    p = GRIDS["small"]()
    a, b = _pair(wd, p, max_cycles=cap)
    try:
        f = wd.wd_rhs(a, p.u0)
        r = _same(wd, a, b, f, tol=1e-12)
        assert r["status"] == wd.WD_E_NOCONV and r["cycles"] == cap
    finally:
        a.close()
        b.close()


def test_device_loop_nonfinite(wd):
    p = GRIDS["tiny"]()
    a, b = _pair(wd, p)
    try:
        f = wd.wd_rhs(a, p.u0)
        f[2, 3, 4] = float("nan")
        r = _same(wd, a, b, f)
        assert r["status"] == wd.WD_E_NONFINITE
        # still usable
        f = wd.wd_rhs(a, p.u0)
        assert _same(wd, a, b, f)["status"] == wd.WD_OK
    finally:
        a.close()
        b.close()


def test_device_loop_diverged(wd):
    p = GRIDS["tiny"]()
    a, b = _pair(wd, p, env={"WD_TEST_CORRECTION_WEIGHT": "4"})
    try:
        f = wd.wd_rhs(a, p.u0)
        r = _same(wd, a, b, f)
        assert r["status"] == wd.WD_E_DIVERGED
    finally:
        a.close()
        b.close()


def test_device_loop_not_used_when_profiling(wd):
    """Conditional bodies cannot hold the profiler's event records: with
    profile on, wd_solve keeps the host loop (no loop kernels launched)."""
    p = GRIDS["small"]()
    a = wd.wd_assemble(p.X, p.Y, p.Z, p.a,
                       wd.default_options(coarsest_max_free=60, device_loop=1, profile=1))
    b = wd.wd_assemble(p.X, p.Y, p.Z, p.a,
                       wd.default_options(coarsest_max_free=60, device_loop=0, profile=1))
    try:
        f = wd.wd_rhs(a, p.u0)
        n0 = wd.wd_launch_count()
        la, ra = wd.wd_solve(a, f, rel_tol=1e-10)
        n1 = wd.wd_launch_count()
        lb, rb = wd.wd_solve(b, f, rel_tol=1e-10)
        n2 = wd.wd_launch_count()
        assert torch.equal(la, lb) and n1 - n0 == n2 - n1
    finally:
        a.close()
        b.close()

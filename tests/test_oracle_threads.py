"""The oracle's parallel loops do not change its arithmetic.

orc.c runs its scatter loops (element assembly, one-point assembly, RHS, D1,
Galerkin, restriction) owner-partitioned by target row: each thread executes
the serial loop in serial order and adds only into rows it owns, so every
entry receives the same terms in the same order as with one thread.  These
tests pin that: one thread and several threads give bitwise equal results on
a ragged grid (odd/even sizes, vertical merging, several coarse levels).
"""
import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def prob():
    return synth.hill(nx=37, ny=22, nz=6, dx=50.0, height=200.0, sigma=300.0, dz0=10.0, r=1.3,
                      a=(1.0, 1.0, 10.0))


def _all(p):
    X, Y, Z, u0 = p.numpy()
    mg = oracle.MG(X, Y, Z, p.a, coarsest_max_free=60)
    f = oracle.rhs(X, Y, Z, u0)
    rng = np.random.default_rng(5)
    r = rng.standard_normal(mg.shape(0))
    out = [oracle.assemble(X, Y, Z, p.a), oracle.assemble_onepoint(X, Y, Z, p.a), f,
           oracle.d1(X, Y, Z, u0), mg.restrict(0, r)]
    out += [mg.K(l) for l in range(mg.nlev)]
    lam, rep = mg.solve(f, tol=1e-10)
    out.append(lam)
    return out, mg.nlev


def test_threads_bitwise(prob):
    n0 = oracle.num_threads()
    try:
        oracle.set_threads(1)
        a, nl = _all(prob)
        oracle.set_threads(max(4, n0))
        b, nl2 = _all(prob)
    finally:
        oracle.set_threads(n0)
    assert nl == nl2 and nl >= 3
    for x, y in zip(a, b):
        assert np.array_equal(x, y)

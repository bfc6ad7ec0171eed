"""The seeded input generator (synth/) builds valid inputs with the stated
recipes (reading R1 of DESIGN.md)."""
import numpy as np
import pytest

import oracle
import synth


def test_levels_geometric():
    z = synth.stretched_levels(15, 10.0, 1.25)
    d = np.diff(z)
    assert d[0] == 10.0
    np.testing.assert_allclose(d[1:] / d[:-1], 1.25, rtol=1e-12)


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_config_mesh_valid(name):
    p = synth.make(name)
    X, Y, Z, u0 = p.numpy()
    assert X.shape == (p.nz + 1, p.ny + 1, p.nx + 1)
    assert u0.shape == (3, p.nz, p.ny, p.nx)
    assert oracle.validate_mesh(X, Y, Z)[0] is None
    # R1: flat top, min terrain 0, first layer dz0 at the highest column
    assert np.ptp(Z[-1]) <= 1e-12 * Z[-1].max() and Z[0].min() == 0
    jm, im = np.unravel_index(np.argmax(Z[0]), Z[0].shape)
    assert abs((Z[1, jm, im] - Z[0, jm, im]) - p.meta["dz0"]) < 1e-9


def test_seeded_reproducible():
    a = synth.small().u0
    b = synth.small().u0
    assert bool((a == b).all())


def test_ridge_terrain_small_instance():
    """The Medium/Paper recipe on a small grid: rms, slope cap, min 0."""
    rng = np.random.default_rng(2)
    zs = synth.fractal_ridges(rng, 201, 201, 30.0, 30.0, 200.0)
    assert float(zs.min()) == 0.0
    g = (zs[:, 2:] - zs[:, :-2]) / 60.0
    assert float(g.abs().max()) <= np.tan(np.radians(35)) + 1e-12


def test_warm_increment_rms():
    p = synth.crop(synth.small(), 0, 0, 128, 128)
    d = synth.warm_increment(p, 4, corr_len=500.0)
    for c in range(2):
        assert abs(float(d[c, 0].pow(2).mean().sqrt()) - 0.5) < 1e-12
        assert bool((d[c] == d[c, 0:1]).all())
    assert not d[2].any()

"""Pin of the planner's inputs (reading C2 of DESIGN.md; "at the
bottom of the grid, the grid spacing is h1 = h2 ... and h3"): h1 = sqrt(dx dy)
from the grid origin, h3 = the layer thicknesses of the column of minimum
terrain height Z(i,j,0), ties resolved to the smallest linear index j n1 + i.
The grids are written out by hand here (no synth/ recipe), with every column's
layers different so that picking the wrong column changes h3."""
import numpy as np

import oracle


def _grid(n1, n2, dx, dy, zs, layers_of):
    """X, Y, Z with Z(i,j,k) = zs[j,i] + sum of the first k thicknesses of
    layers_of(i, j)"""
    n3 = len(layers_of(0, 0)) + 1
    X = np.zeros((n3, n2, n1))
    Y = np.zeros((n3, n2, n1))
    Z = np.zeros((n3, n2, n1))
    for j in range(n2):
        for i in range(n1):
            X[:, j, i] = 7.0 + i * dx
            Y[:, j, i] = -3.0 + j * dy
            Z[0, j, i] = zs[j, i]
            for k, t in enumerate(layers_of(i, j)):
                Z[k + 1, j, i] = Z[k, j, i] + t
    return X, Y, Z


def _layers(i, j):
    # thicknesses that identify the column: layer k of column (i,j) is
    # (k + 1) * (1 + i/10 + j/100)
    return [(k + 1) * (1.0 + i / 10.0 + j / 100.0) for k in range(4)]


def test_minimum_column_and_h1():
    n1, n2 = 6, 5
    zs = np.full((n2, n1), 50.0)
    zs[3, 4] = 12.5            # unique minimum at (i, j) = (4, 3)
    X, Y, Z = _grid(n1, n2, 30.0, 120.0, zs, _layers)
    h1, h3 = oracle.planner_inputs(X, Y, Z)
    assert h1 == np.sqrt(30.0 * 120.0)      # geometric mean of dx, dy (C2)
    np.testing.assert_array_equal(h3, np.diff(Z[:, 3, 4]))
    # hand value: column (4, 3) has thicknesses (k+1) * 1.43
    np.testing.assert_allclose(h3, [1.43, 2.86, 4.29, 5.72], rtol=1e-14)


def test_ties_take_smallest_linear_index():
    n1, n2 = 6, 5
    zs = np.full((n2, n1), 50.0)
    for (i, j) in [(5, 1), (2, 3), (0, 4)]:   # linear indices 11, 20, 24
        zs[j, i] = -4.0
    X, Y, Z = _grid(n1, n2, 25.0, 25.0, zs, _layers)
    h1, h3 = oracle.planner_inputs(X, Y, Z)
    assert h1 == 25.0
    np.testing.assert_allclose(h3, [(k + 1) * 1.51 for k in range(4)], rtol=1e-14)
    # the same grid with the first tie removed picks the next one, (2, 3)
    zs[1, 5] = 50.0
    X, Y, Z = _grid(n1, n2, 25.0, 25.0, zs, _layers)
    _, h3 = oracle.planner_inputs(X, Y, Z)
    np.testing.assert_allclose(h3, [(k + 1) * 1.23 for k in range(4)], rtol=1e-14)


def test_minimum_at_origin_and_last_node():
    n1, n2 = 4, 4
    zs = np.arange(n1 * n2, dtype=float).reshape(n2, n1)   # minimum at linear index 0
    X, Y, Z = _grid(n1, n2, 10.0, 10.0, zs, _layers)
    _, h3 = oracle.planner_inputs(X, Y, Z)
    np.testing.assert_allclose(h3, [(k + 1) * 1.0 for k in range(4)], rtol=1e-14)
    zs = -zs                                                   # minimum at the last node
    X, Y, Z = _grid(n1, n2, 10.0, 10.0, zs, _layers)
    _, h3 = oracle.planner_inputs(X, Y, Z)
    np.testing.assert_allclose(h3, [(k + 1) * 1.33 for k in range(4)], rtol=1e-14)

"""Checks of the shared input generator (gen/): the quadrature used for the
input cell averages is exact through degree 5 (R20), meshes tile the box."""
import itertools
import math

import numpy as np
import pytest

import gen


@pytest.mark.parametrize("d", [2, 3])
def test_average_rule_exact_degree5(d):
    bary, w = gen._rule(d)
    assert abs(w.sum() - 1.0) < 1e-15
    # reference simplex: vertices 0, e_1, .., e_d → points = bary[:, 1:]
    P = bary[:, 1:]
    for e in itertools.product(range(6), repeat=d):
        if sum(e) > 5:
            continue
        val = np.sum(w * np.prod(P ** np.array(e), axis=1))
        exact = math.factorial(d) * np.prod([math.factorial(k) for k in e]) / math.factorial(sum(e) + d)
        assert abs(val - exact) < 1e-14


@pytest.mark.parametrize("d,n", [(2, 5), (3, 3)])
def test_box_mesh_counts_and_volume(d, n):
    for periodic in (True, False):
        nodes, cells, period = gen.box_mesh(d, n, periodic, 0.2 if d == 2 else 0.1, 1)
        assert cells.shape == ((2 if d == 2 else 6) * n ** d, d + 1)
        assert nodes.shape[0] == (n if periodic else n + 1) ** d
        X = gen.unwrap_cells(nodes, cells, period)
        vol = np.abs(np.linalg.det(X[:, 1:] - X[:, :1])) / math.factorial(d)
        assert abs(vol.sum() - 1.0) < 1e-12 and vol.min() > 0.2 / n ** d / math.factorial(d)


def test_configs_shapes():
    w = gen.make("C1")
    assert w["cells"].shape == (512, 3) and w["avgs"].shape == (512, 4)
    # vortex density bounds (R21)
    assert 0.49 < w["avgs"][:, 0].min() and w["avgs"][:, 0].max() <= 1.0
    # constant IC -> exactly constant averages (same ops per cell)
    nodes, cells, period = gen.box_mesh(3, 3, True)
    a = gen.cell_averages(nodes, cells, period, lambda P: np.full((P.shape[0], 1), 0.1), 1)
    assert np.all(a == a[0])

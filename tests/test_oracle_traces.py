"""Pins of the face-trace oracle."""
import math
from itertools import product

import numpy as np
import pytest

import gen
from oracle import reconstruct as R
from oracle import traces as TR
from oracle.mesh import OracleMesh


@pytest.mark.parametrize("d,M", [(2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3)])
def test_face_rule_exact_to_degree_2M_plus_1(d, M):
    """Σ_q w_q Π λ_a^{k_a} = (d−1)! Π k_a! / (|k| + d − 1)!  (Dirichlet average over the
    (d−1)-simplex) for every |k| ≤ 2M+1 — and fails at a higher degree."""
    lam, w = TR.face_rule(d, M)
    assert abs(w.sum() - 1) < 1e-15 and np.all(w > 0)
    assert np.allclose(lam.sum(axis=1), 1.0, atol=1e-15) and np.all(lam >= 0)
    for k in product(range(2 * M + 2), repeat=d):
        if sum(k) > 2 * M + 1:
            continue
        exact = math.factorial(d - 1) * math.prod(math.factorial(x) for x in k) / math.factorial(sum(k) + d - 1)
        got = float(np.sum(w * np.prod(lam ** np.array(k), axis=1)))
        assert abs(got - exact) <= 1e-14 * max(1.0, exact), (k, got, exact)
    k = (2 * M + 2,) + (0,) * (d - 1)
    exact = math.factorial(d - 1) * math.factorial(2 * M + 2) / math.factorial(2 * M + 2 + d - 1)
    got = float(np.sum(w * lam[:, 0] ** (2 * M + 2)))
    assert abs(got - exact) > 1e-13


def _poly_case(d, M, n, seed):
    nodes, cells, _ = gen.box_mesh(d, n, False, 0.15, seed)
    m = OracleMesh(nodes, cells, None, M)
    rng = np.random.default_rng(seed)
    exps = [e for e in product(range(M + 1), repeat=d) if sum(e) <= M]
    coef = rng.standard_normal((2, len(exps)))
    def p(x):
        return np.stack([sum(c * np.prod(x ** np.array(e), axis=-1) for c, e in zip(coef[v], exps))
                         for v in range(2)], axis=-1)
    Q = gen.polynomial_averages(nodes, cells, [lambda x, v=v: p(x)[..., v] for v in range(2)])[m.perm]
    return m, Q, p


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2)])
def test_traces_of_reproduced_polynomials(d, M):
    """Polynomial data of degree ≤ M is reproduced exactly by P_opt on interior cells
    (pinned in test_oracle_reconstruct), so the traces of P_opt must equal the
    polynomial at the physical face points; both cells of an interior face agree.
    (The blended w differs from P_opt by the nonlinear weights, O(1/λ0).)"""
    m, Q, p = _poly_case(d, M, 7 if d == 2 else 4, 5)
    centre = m.bary.mean(axis=0)
    inner = np.argsort(np.linalg.norm(m.bary - centre, axis=1))[:6]
    for i in inner:
        w = R.reconstruct_cell(m, int(i), Q, M)["popt"]
        tr = TR.cell_traces(m, int(i), w, M)
        for f in range(d + 1):
            x = TR.face_points(m, int(i), f, M)
            assert np.abs(tr[f] - p(x)).max() <= 1e-10 * max(1.0, np.abs(p(x)).max())
            j = int(m.nbr[i][f])
            if j < 0:
                continue
            fj = [g for g in range(d + 1) if int(m.nbr[j][g]) == int(i)][0]
            assert np.allclose(TR.face_points(m, j, fj, M), x, atol=1e-14)   # same points, same order

"""Pins for oracle/basis.py against the paper and against independent mathematics.

Every check here is computed by a route different from the oracle's own: the
Dirichlet monomial formula is checked against sympy.integrate with explicit
limits; orthonormality and Σ against Gauss quadrature on the collapsed square
/ cube with sympy-lambdified derivatives; Σ on linear and quadratic
polynomials against hand-derived closed forms.
"""
import itertools
import math

import numpy as np
import pytest
import sympy as sp

from oracle import basis as B


def test_n_modes_paper_counts(golden):
    # Eq. cwenoM evaluated at the paper's runs: DOF = N_E * M(M,d)
    for row in golden["dof"]:
        assert row["N_E"] * B.n_modes(row["M"], row["d"]) == row["DOF"], row["cite"]
    for row in golden["stencil_size"]:
        assert row["d"] * B.n_modes(row["M"], row["d"]) == row["n_e"], row["cite"]
    assert [B.n_modes(M, 2) for M in range(1, 5)] == [3, 6, 10, 15]
    assert [B.n_modes(M, 3) for M in range(1, 5)] == [4, 10, 20, 35]


@pytest.mark.parametrize("exps", [(0, 0), (1, 0), (2, 3), (4, 1), (0, 0, 0), (1, 2, 0), (2, 1, 3), (0, 0, 5)])
def test_dirichlet_formula_vs_sympy_integrate(exps):
    x, y, z = sp.symbols("x y z")
    if len(exps) == 2:
        f = x ** exps[0] * y ** exps[1]
        ref = sp.integrate(sp.integrate(f, (x, 0, 1 - y)), (y, 0, 1))
    else:
        f = x ** exps[0] * y ** exps[1] * z ** exps[2]
        ref = sp.integrate(sp.integrate(sp.integrate(f, (x, 0, 1 - y - z)), (y, 0, 1 - z)), (z, 0, 1))
    assert B.monomial_integral(exps) == ref


def _collapsed_rule(d, n):
    """Gauss-Legendre on [0,1]^d with the Duffy collapse and its Jacobian."""
    g, w = np.polynomial.legendre.leggauss(n)
    g = (g + 1) / 2
    w = w / 2
    pts, wts = [], []
    for idx in itertools.product(range(n), repeat=d):
        u = [g[k] for k in idx]
        wt = np.prod([w[k] for k in idx])
        if d == 2:
            eta = u[1]
            xi = u[0] * (1 - u[1])
            pts.append((xi, eta)); wts.append(wt * (1 - u[1]))
        else:
            zeta = u[2]
            eta = u[1] * (1 - u[2])
            xi = u[0] * (1 - u[1]) * (1 - u[2])
            pts.append((xi, eta, zeta)); wts.append(wt * (1 - u[1]) * (1 - u[2]) ** 2)
    return np.array(pts), np.array(wts)


def _lamb(expr, d):
    f = sp.lambdify(B.syms(d), expr, "numpy")
    return lambda P: np.broadcast_to(np.asarray(f(*P.T), dtype=float), (P.shape[0],))


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3)])
def test_orthonormal_by_quadrature(d, M):
    psis = B.dubiner_sympy(d, M)
    P, W = _collapsed_rule(d, M + 3)
    vals = np.array([_lamb(p, d)(P) for p in psis])
    G = (vals * W) @ vals.T
    assert np.abs(G - np.eye(len(psis))).max() < 1e-12
    assert abs(float(psis[0]) - math.sqrt(math.factorial(d))) < 1e-15
    assert B.psi1(d) == math.sqrt(math.factorial(d))


@pytest.mark.parametrize("d,M", [(2, 2), (3, 2)])
def test_mean_zero_and_p1_span_exact(d, M):
    psis = B.dubiner_sympy(d, M)
    X = B.syms(d)
    for p in psis[1:]:
        assert sp.simplify(B.integrate_TE(p, d)) == 0
    # the first d+1 functions are exactly the polynomials of degree <= 1 (R8)
    for l, p in enumerate(psis):
        deg = sp.Poly(p, *X).total_degree()
        assert (deg <= 1) == (l <= d)
    J = sp.Matrix([[sp.diff(psis[l], v) for v in X] for l in range(1, d + 1)])
    assert J.det() != 0


def _sigma_quadrature(d, M):
    psis = B.dubiner_sympy(d, M)
    X = B.syms(d)
    P, W = _collapsed_rule(d, M + 2)
    alphas = [a for a in itertools.product(range(M + 1), repeat=d) if 1 <= sum(a) <= M]
    D = np.zeros((len(alphas), len(psis), len(W)))
    for t, a in enumerate(alphas):
        for l, p in enumerate(psis):
            e = p
            for v, k in zip(X, a):
                e = sp.diff(e, v, k)
            D[t, l] = _lamb(e, d)(P)
    return np.einsum("tlq,tmq,q->lm", D, D, W)


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_sigma_vs_quadrature_and_structure(d, M):
    S = B.sigma_numeric(d, M)
    Sq = _sigma_quadrature(d, M)
    assert np.abs(S - Sq).max() < 1e-9 * np.abs(Sq).max()
    assert np.array_equal(S, S.T)
    assert np.all(S[0] == 0) and np.all(S[:, 0] == 0)          # ψ_1 constant
    ev = np.linalg.eigvalsh(S[1:, 1:])
    assert ev.min() > 0                                          # σ = 0 iff constant


@pytest.mark.parametrize("d,M", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_sigma_linear_closed_form(d, M):
    # For p ∈ ℙ1 only first derivatives survive: σ = |T_E| |∇p|^2, |T_E| = 1/d!.
    rng = np.random.default_rng(7)
    psis = B.dubiner_sympy(d, M)
    X = B.syms(d)
    c = rng.standard_normal(d + 1)
    p = sum(float(c[l]) * psis[l] for l in range(d + 1))
    grad = np.array([float(sp.diff(p, v)) for v in X])
    full = np.zeros(len(psis)); full[: d + 1] = c
    sigma = full @ B.sigma_numeric(d, M) @ full
    assert abs(sigma - grad @ grad / math.factorial(d)) < 1e-12 * (grad @ grad)


def test_sigma_quadratic_hand_value():
    # p = ξ² on T_E (2D, M=2): Σ_α ∫ (∂^α p)^2 = ∫ (2ξ)^2 + ∫ 2^2 = 4/12 + 4/2 = 7/3
    d, M = 2, 2
    psis = B.dubiner_sympy(d, M)
    xi = B.XI
    coef = np.array([float(B.integrate_TE(xi ** 2 * p, d)) for p in psis])   # orthonormal projection
    sigma = coef @ B.sigma_numeric(d, M) @ coef
    assert abs(sigma - 7.0 / 3.0) < 1e-12

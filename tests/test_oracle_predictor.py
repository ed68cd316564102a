"""Pins for oracle/predictor.py (the local space-time Galerkin predictor)
against what the paper and mathematics fix (no GPU).

* Space-time basis: 𝓛 = ℳ(M, d+1) nodal functions, ℳ(M, d) of them at
  τ = 0 (SPEC's example: 𝓛 = 10 with 6 τ = 0 nodes for M = 2, d = 2); Lagrange
  property θ_l(ξ̃_k) = δ_kl.
* Matrices of Eq. cgPDE, exact: K_τ·1 = 0 (∂τ of a constant);
  K_τ + K_τᵀ = B(1) − B(0) with B(t)_kl = ∫_{T_E} θ_kθ_l at τ = t (integration by
  parts in τ, evaluated independently by substitution); M symmetric positive
  definite with Σ_kl M_kl = |T_E| (partition of unity); the unknown-node block of
  K_τ is invertible (R33).
* Constant state: H = 0, so the predictor is the constant (Eq. PDExi2).
* Contact wave (ρ = polynomial of degree ≤ M, u and p constant): the Euler flux is
  affine in the state on this family and the exact solution q(x − u t) is a
  space-time polynomial of degree M, so the Galerkin predictor reproduces it at
  every node (SPEC S:392's linear-advection case, on the Euler system).
* Pressure and energy fluxes: ρ constant, u and p linear, M = 3 → every flux
  component is a polynomial of degree ≤ 3, the nodal interpolant F_h is exact,
  and ∂q_h/∂τ(ξ, 0)/Δt → −∇·F(q(x)) as Δt → 0, compared with sympy's symbolic
  divergence of the Euler flux.
* Picard iteration on smooth data converges within the 2(M+1) cap.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest
import sympy as sp

from oracle import basis as B
from oracle import predictor as PR


@pytest.mark.parametrize("d,M", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_space_time_matrices_exact(d, M):
    S = PR.st_matrices(d, M)
    L = len(S["nodes"])
    assert L == B.n_modes(M, d + 1)
    assert int(S["known"].sum()) == B.n_modes(M, d)
    if (d, M) == (2, 2):
        assert (L, int(S["known"].sum())) == (10, 6)
    # Lagrange property (exact)
    C, monos = S["C"], S["monos"]
    for k, x in enumerate(S["nodes"]):
        for l in range(L):
            v = sum(C[j][l] * math.prod(xc ** ac for xc, ac in zip(x, a)) for j, a in enumerate(monos))
            assert v == (1 if k == l else 0)
    Kt, Mm = S["Kt_exact"], S["M_exact"]
    # K_τ·1 = 0
    for k in range(L):
        assert sum(Kt[k]) == 0
    # K_τ + K_τᵀ = B(1) − B(0), B(t) by substituting τ = t and integrating over T_E
    def te_int(e):
        return Fraction(math.prod(math.factorial(x) for x in e), math.factorial(sum(e) + len(e)))

    def Bt(t):
        out = [[Fraction(0)] * L for _ in range(L)]
        for k in range(L):
            for l in range(L):
                s = Fraction(0)
                for i, a in enumerate(monos):
                    if C[i][k] == 0:
                        continue
                    for j, b in enumerate(monos):
                        if C[j][l] == 0:
                            continue
                        s += C[i][k] * C[j][l] * Fraction(t) ** (a[-1] + b[-1]) * te_int(
                            tuple(x + y for x, y in zip(a[:-1], b[:-1])))
                out[k][l] = s
        return out
    B1, B0 = Bt(1), Bt(0)
    for k in range(L):
        for l in range(L):
            assert Kt[k][l] + Kt[l][k] == B1[k][l] - B0[k][l]
            assert Mm[k][l] == Mm[l][k]
    assert sum(sum(r) for r in Mm) == Fraction(1, math.factorial(d))
    assert np.all(np.linalg.eigvalsh(S["Mm"]) > 0)
    unk = ~S["known"]
    assert np.linalg.matrix_rank(S["Kt"][np.ix_(unk, unk)]) == int(unk.sum())


def _cell(d, seed=0):
    rng = np.random.default_rng(seed)
    if d == 2:
        X = np.array([[0.0, 0.0], [0.05, 0.0], [0.0, 0.05]])
    else:
        X = np.array([[0.0, 0.0, 0.0], [0.05, 0.0, 0.0], [0.0, 0.05, 0.0], [0.0, 0.0, 0.05]])
    X = X + rng.uniform(-0.008, 0.008, X.shape) + 0.3
    return X


def _rule(d, n=7):
    g, w = np.polynomial.legendre.leggauss(n)
    g, w = (g + 1) / 2, w / 2
    pts, wts = [], []
    for idx in itertools.product(range(n), repeat=d):
        u = [g[k] for k in idx]
        wt = np.prod([w[k] for k in idx])
        if d == 2:
            pts.append((u[0] * (1 - u[1]), u[1])); wts.append(wt * (1 - u[1]))
        else:
            pts.append((u[0] * (1 - u[1]) * (1 - u[2]), u[1] * (1 - u[2]), u[2]))
            wts.append(wt * (1 - u[1]) * (1 - u[2]) ** 2)
    return np.array(pts), np.array(wts)


def _project(X, f, d, M):
    """Orthonormal Dubiner projection of f(x(ξ)) on the cell: w [V][ℳ] (exact for
    polynomials of degree ≤ M; independent of the predictor's node evaluation)."""
    P, W = _rule(d)
    x = X[0] + P @ (X[1:] - X[0])
    psi = np.array([np.broadcast_to(np.asarray(sp.lambdify(B.syms(d), p, "numpy")(*P.T), float), (len(P),))
                    for p in B.dubiner_sympy(d, M)])
    return ((psi * W) @ f(x)).T


def _node_xt(X, S, dt):
    d = X.shape[1]
    nodes = np.array([[float(v) for v in x] for x in S["nodes"]])
    x = X[0] + nodes[:, :d] @ (X[1:] - X[0])
    return x, nodes[:, d] * dt


@pytest.mark.parametrize("d,M", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_constant_state(d, M):
    X = _cell(d)
    q0 = np.array([1.2] + [0.3, -0.2, 0.1][:d] + [3.0])
    w = _project(X, lambda x: np.tile(q0, (x.shape[0], 1)), d, M)
    r = PR.predict_cell(X, w, 0.01, M)
    assert r["converged"] and r["admissible"]
    assert np.abs(r["q"] - q0).max() < 1e-12 * np.abs(q0).max()    # κ(K_τ¹¹) ≤ 5e4 amplifies rounding


@pytest.mark.parametrize("d,M", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_contact_wave_exact(d, M):
    """ρ(x, t) = ρ_0(x − u t), u, p constant: the predictor equals the exact
    space-time polynomial at every node (affine flux on this family)."""
    X = _cell(d, 1)
    g = PR.GAMMA
    u = np.array([0.7, -0.4, 0.25][:d])
    p0 = 1.3
    a = np.array([0.9, -1.7, 0.6][:d])
    b = np.array([-0.5, 0.8, 1.1][:d])
    c = np.array([0.4, 0.3, -0.9][:d])

    def rho(x):
        s = x - 0.3
        r = 1.0 + s @ a
        if M >= 2:
            r = r + 2.0 * (s @ b) ** 2
        if M >= 3:
            r = r + 5.0 * (s @ c) ** 3
        return r

    def state(x):
        r = rho(x)
        return np.column_stack([r] + [r * u[k] for k in range(d)] + [p0 / (g - 1) + 0.5 * r * (u @ u)])
    w = _project(X, state, d, M)
    dt = 0.02
    res = PR.predict_cell(X, w, dt, M)
    assert res["converged"] and res["admissible"] and res["iters"] <= M + 2
    x, t = _node_xt(X, PR.st_matrices(d, M), dt)
    exact = state(x - t[:, None] * u[None, :])
    assert np.abs(res["q"] - exact).max() < 1e-11 * np.abs(exact).max()


def test_time_derivative_is_minus_divergence_of_euler_flux():
    """d = 2, M = 3, ρ const, u and p linear: F is cubic in x, F_h exact; the
    predictor's ∂q_h/∂τ at τ = 0 divided by Δt tends to −∇·F(q(x)) (Eq. PDExi2)."""
    d, M = 2, 3
    X = _cell(d, 2)
    g = PR.GAMMA
    xs, ys = sp.symbols("x y")
    rho = sp.Rational(13, 10)
    u = [sp.Rational(1, 2) + sp.Rational(3, 5) * (xs - sp.Rational(3, 10)) - sp.Rational(2, 5) * (ys - sp.Rational(3, 10)),
         -sp.Rational(3, 10) + sp.Rational(1, 5) * (xs - sp.Rational(3, 10)) + sp.Rational(7, 10) * (ys - sp.Rational(3, 10))]
    p = 2 + sp.Rational(4, 5) * (xs - sp.Rational(3, 10)) - sp.Rational(3, 5) * (ys - sp.Rational(3, 10))
    E = p / (g - 1) + rho * (u[0] ** 2 + u[1] ** 2) / 2
    q = [rho, rho * u[0], rho * u[1], E]
    F = [[rho * u[a], rho * u[a] * u[0] + (p if a == 0 else 0), rho * u[a] * u[1] + (p if a == 1 else 0),
          u[a] * (E + p)] for a in range(2)]
    divF = [sp.diff(F[0][v], xs) + sp.diff(F[1][v], ys) for v in range(4)]
    qf = [sp.lambdify((xs, ys), e, "numpy") for e in q]
    df = [sp.lambdify((xs, ys), e, "numpy") for e in divF]

    def state(x):
        return np.column_stack([np.broadcast_to(np.asarray(f(x[:, 0], x[:, 1]), float), (x.shape[0],)) for f in qf])
    w = _project(X, state, d, M)
    S = PR.st_matrices(d, M)
    known = S["known"]
    x0, _ = _node_xt(X, S, 0.0)
    want = -np.column_stack([np.asarray(f(x0[:, 0], x0[:, 1]), float) * np.ones(len(x0)) for f in df])[known]
    nodes0 = np.array([[float(v) for v in xx] for xx in S["nodes"]])[known]
    errs = []
    for dt in (1e-3, 1e-4):
        r = PR.predict_cell(X, w, dt, M)
        # ∂/∂τ of Σ_l θ_l q̂_l at the τ = 0 nodes, exactly from the monomial coefficients
        C = np.array([[float(v) for v in row] for row in S["C"]])
        dP = np.array([[a[-1] * (1.0 if a[-1] == 1 else 0.0) * np.prod([xx ** e for xx, e in zip(pt[:d], a[:d])])
                        for a in S["monos"]] for pt in nodes0])   # ∂τ τ^k at τ=0: only k = 1 survives
        dq = dP @ C @ r["q"] / dt
        errs.append(np.abs(dq - want).max() / np.abs(want).max())
    assert max(errs) < 1e-6, errs      # −∇·F to O(Δt) + rounding (a wrong flux term: O(1))


def test_picard_converges_on_smooth_data():
    for d, M in [(2, 3), (3, 2)]:
        X = _cell(d, 3)

        def state(x):
            r = 1.0 + 0.2 * np.sin(3 * x[:, 0]) * np.cos(2 * x[:, 1])
            vel = [0.3 * np.cos(x[:, 1]), -0.2 * np.sin(x[:, 0]), 0.1 + 0 * x[:, 0]][:d]
            pp = 1.0 + 0.1 * np.cos(x[:, 0] + x[:, 1])
            return np.column_stack([r] + [r * v for v in vel] + [pp / 0.4 + 0.5 * r * sum(v * v for v in vel)])
        w = _project(X, state, d, M)
        r = PR.predict_cell(X, w, 0.02, M)     # CFL ≈ 0.02·(|u|+c)/0.05 ≈ 0.5/d
        assert r["converged"] and r["admissible"] and r["iters"] <= 2 * (M + 1)

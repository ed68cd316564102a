"""Oracle: orthonormal Dubiner basis on T_E and the oscillation matrix Σ, exact (sympy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Basis (Eq. recpolydef): "orthogonal Dubiner-type basis functions
  ψ_l(ξ) on the reference element T_E".  Reading R8: orthonormal on T_E
  (∫_{T_E} ψ_l ψ_m = δ_lm), graded order
      2D: for n: for q in 0..n: p = n-q          -> ψ_{pq}
      3D: for n: for r in 0..n: for q in 0..n-r: p = n-q-r -> ψ_{pqr}
  built from the collapsed-coordinate Jacobi product (Dubiner / Sherwin-
  Karniadakis) and homogenised into polynomials.
* Σ: Σ_lm = Σ_{1 ≤ |α| ≤ M} ∫_{T_E} ∂^α ψ_l ∂^α ψ_m; each multi-
  index counted once (R9).
* ℳ(M, d) = (1/d!) Π_{l=1..d} (M+l)  (Eq. cwenoM).

Integrals over T_E are done exactly with the Dirichlet monomial formula
    ∫_{T_E} ξ^a η^b [ζ^c] = a! b! [c!] / (a+b[+c]+d)!
which tests/test_oracle_basis.py pins against sympy.integrate.
"""
from __future__ import annotations

import functools
import itertools
import math

import numpy as np
import sympy as sp

XI, ETA, ZETA = sp.symbols("xi eta zeta")


def n_modes(M: int, d: int) -> int:
    """ℳ(M,d)."""
    num = 1
    for l in range(1, d + 1):
        num *= (M + l)
    return num // math.factorial(d)


def mode_indices(M: int, d: int):
    """Graded ordering R8: list of (p,q) or (p,q,r)."""
    out = []
    for n in range(M + 1):
        if d == 2:
            for q in range(n + 1):
                out.append((n - q, q))
        else:
            for r in range(n + 1):
                for q in range(n - r + 1):
                    out.append((n - q - r, q, r))
    return out


def _homog_jacobi(n, a, b, num, den):
    """P_n^{(a,b)}(num/den) * den^n as a polynomial (exact)."""
    t = sp.Symbol("t")
    P = sp.Poly(sp.jacobi(n, a, b, t), t)
    expr = 0
    for (k,), c in P.terms():
        expr += c * num ** k * den ** (n - k)
    return sp.expand(expr)


@functools.lru_cache(maxsize=None)
def dubiner_sympy(d: int, M: int):
    """Orthonormal Dubiner functions on T_E as exact sympy polynomials."""
    psis = []
    for idx in mode_indices(M, d):
        if d == 2:
            p, q = idx
            f1 = _homog_jacobi(p, 0, 0, 2 * XI + ETA - 1, 1 - ETA)
            f2 = sp.expand(sp.jacobi(q, 2 * p + 1, 0, 2 * ETA - 1))
            c = sp.sqrt(sp.Integer((2 * p + 1) * (2 * p + 2 * q + 2)))
            psis.append(sp.expand(c * f1 * f2))
        else:
            p, q, r = idx
            f1 = _homog_jacobi(p, 0, 0, 2 * XI + ETA + ZETA - 1, 1 - ETA - ZETA)
            f2 = _homog_jacobi(q, 2 * p + 1, 0, 2 * ETA + ZETA - 1, 1 - ZETA)
            f3 = sp.expand(sp.jacobi(r, 2 * p + 2 * q + 2, 0, 2 * ZETA - 1))
            c = sp.sqrt(sp.Integer((2 * p + 1) * (2 * p + 2 * q + 2) * (2 * p + 2 * q + 2 * r + 3)))
            psis.append(sp.expand(c * f1 * f2 * f3))
    return tuple(psis)


def syms(d):
    return (XI, ETA) if d == 2 else (XI, ETA, ZETA)


def monomial_integral(exps) -> sp.Rational:
    """∫_{T_E} Π ξ_a^{e_a} = Π e_a! / (Σe + d)!  (Dirichlet integral)."""
    d = len(exps)
    num = 1
    for e in exps:
        num *= math.factorial(e)
    return sp.Rational(num, math.factorial(sum(exps) + d))


def integrate_TE(expr, d):
    """Exact ∫_{T_E} expr for a polynomial expr."""
    P = sp.Poly(sp.expand(expr), *syms(d))
    total = sp.Integer(0)
    for exps, c in P.terms():
        total += c * monomial_integral(exps)
    return sp.nsimplify(sp.simplify(total)) if total.free_symbols else sp.simplify(total)


def multi_indices(d, lo, hi):
    return [a for a in itertools.product(range(hi + 1), repeat=d) if lo <= sum(a) <= hi]


@functools.lru_cache(maxsize=None)
def sigma_sympy(d: int, M: int):
    """Σ_lm exactly, as a sympy Matrix."""
    psis = dubiner_sympy(d, M)
    X = syms(d)
    n = len(psis)
    alphas = multi_indices(d, 1, M)
    derivs = []
    for psi in psis:
        ds = []
        for a in alphas:
            e = psi
            for var, k in zip(X, a):
                if k:
                    e = sp.diff(e, var, k)
            ds.append(sp.expand(e))
        derivs.append(ds)
    S = sp.zeros(n, n)
    for l in range(n):
        for m in range(l, n):
            tot = sp.Integer(0)
            for t in range(len(alphas)):
                if derivs[l][t] == 0 or derivs[m][t] == 0:
                    continue
                P = sp.Poly(sp.expand(derivs[l][t] * derivs[m][t]), *X)
                for exps, c in P.terms():
                    tot += c * monomial_integral(exps)
            tot = sp.radsimp(sp.expand(tot))
            S[l, m] = tot
            S[m, l] = tot
    return S


@functools.lru_cache(maxsize=None)
def basis_numeric(d: int, M: int):
    """fp64 monomial form of the basis: (exponents [K,d] int, coeff [ℳ,K] float)."""
    psis = dubiner_sympy(d, M)
    X = syms(d)
    exps = multi_indices(d, 0, M)
    col = {e: k for k, e in enumerate(exps)}
    C = np.zeros((len(psis), len(exps)))
    for l, psi in enumerate(psis):
        for e, c in sp.Poly(psi, *X).terms():
            C[l, col[e]] = float(sp.N(c, 30))
    return np.array(exps, dtype=np.int64), C


@functools.lru_cache(maxsize=None)
def sigma_numeric(d: int, M: int) -> np.ndarray:
    S = sigma_sympy(d, M)
    return np.array([[float(sp.N(S[i, j], 30)) for j in range(S.shape[1])] for i in range(S.shape[0])])


def psi1(d: int) -> float:
    """The constant basis function ψ_1 = 1/sqrt(|T_E|) = sqrt(d!)."""
    return math.sqrt(math.factorial(d))

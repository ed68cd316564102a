"""Oracle: the element-local space-time Galerkin predictor (ADER, Eulerian), literally.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Paper §2.2;
SURVEY §8(f) NEXT-2.  One cell at a time, exact rational matrices (sympy), the
Picard iteration in fp64 numpy in the paper's notation.

Steps (paper order), readings R32-R36 of DESIGN.md:
 1. Space-time reference element T_E × [0,1], coordinates ξ̃ = (ξ, τ).
    τ = (t − tⁿ)/Δt (Eq. timestep), so ∂τ/∂t = 1/Δt and the PDE reads
    ∂Q/∂τ + Δt H(Q) = 0 (Eq. PDExi2) with H(Q) = (∂ξ/∂x)ᵀ ∇_ξ · F(Q) on a fixed
    mesh (Eq. Hterm, mesh velocity 0: the ∂ξ/∂t term vanishes).
 2. Nodal space-time basis θ_l, l < 𝓛 = ℳ(M, d+1) (Eq. qh): Lagrange
    polynomials of total degree M in (ξ, τ) through the nodes of the uniform
    lattice of the (d+1)-simplex {ξ_a ≥ 0, τ ≥ 0, Σξ + τ ≤ 1} with spacing 1/M
    (R32; the paper cites an external node list).  Its τ = 0 nodes are the
    degree-M spatial lattice: the KNOWN degrees of freedom q̂⁰.
 3. K_τ[k][l] = ∫∫ θ_k ∂θ_l/∂τ and M[k][l] = ∫∫ θ_k θ_l over T_E × [0,1]
    (Eq. cgPDE), exact rationals.
 4. F_h = θ_l F(q̂_l), H_h = θ_l H(q̂_l) (Eq. PDEterm): the nodal flux
    interpolant; Ĥ_l = ∇_x · F_h at node l = Σ_m Σ_b (∂ξ_b/∂x_a) ∂θ_m/∂ξ_b(ξ̃_l) F_a(q̂_m)
    (R34).
 5. Picard iteration (Eq. CGfinal):
        K_τ¹ q̂¹^{r+1} = −Δt M Ĥ^r − K_τ⁰ q̂⁰,
    K_τ = (K_τ⁰ | K_τ¹) split by columns into known / unknown nodes; the test
    functions are the θ_k of the UNKNOWN nodes, which makes the system square
    (R33).  Initial guess: q̂_l = w(ξ_l) at every node (constant in τ, R35).
    Stop when max |q̂^{r+1} − q̂^r| ≤ 1e-12·max(1, max|q̂⁰|) or after 2(M+1)
    iterations; at the cap the cell still counts as converged when the last update
    is ≤ 1e-8·max(1, max|q̂⁰|) (R35).
 6. Euler equations, conserved q = (ρ, ρu_1..ρu_d, E),
    F_a = (ρu_a, ρu_a u + p e_a, u_a (E + p)), p = (γ−1)(E − ½ρ|u|²).
"""
from __future__ import annotations

import functools
import itertools
import math
from fractions import Fraction

import numpy as np
import sympy as sp

from .basis import dubiner_sympy, n_modes, syms

GAMMA = 1.4      # P:754 (ideal gas, γ = 1.4)
TOL = 1e-12      # R35
TOL_CAP = 1e-8   # R35: acceptable last update at the iteration cap
MAXIT_FACTOR = 2  # cap 2(M+1) (R35)


def st_nodes(d, M):
    """Uniform lattice of the (d+1)-simplex, spacing 1/M: Fractions [(ξ_1..ξ_d, τ)].
    Order: known (τ = 0) nodes first, each group by the integer tuple ascending."""
    pts = [e for e in itertools.product(range(M + 1), repeat=d + 1) if sum(e) <= M]
    pts.sort(key=lambda e: (e[d] > 0, e[d], e))
    return [tuple(Fraction(x, M) for x in e) for e in pts]


def _monos(n, M):
    return [e for e in itertools.product(range(M + 1), repeat=n) if sum(e) <= M]


def _te_int(exps):
    """∫_{T_E} Π ξ_a^{e_a} = Π e_a! / (Σe + d)!  (Dirichlet)."""
    num = 1
    for e in exps:
        num *= math.factorial(e)
    return Fraction(num, math.factorial(sum(exps) + len(exps)))


def _prism_int(e):
    """∫_{T_E × [0,1]} ξ^{e_ξ} τ^{e_τ}."""
    return _te_int(e[:-1]) * Fraction(1, e[-1] + 1)


@functools.lru_cache(maxsize=None)
def st_matrices(d, M):
    """Exact space-time matrices of (d, M): dict of Fractions-based numpy object arrays
    and float copies:
        nodes [𝓛][d+1], known (bool [𝓛]), C [n_mono][𝓛] (θ_l = Σ_α C[α][l] ξ̃^α),
        Kt [𝓛][𝓛], Mm [𝓛][𝓛], D [d][𝓛][𝓛] (D[b][l][m] = ∂θ_m/∂ξ_b at node l),
        Phi [𝓛][ℳ] (ψ_m at the spatial part of node l, float)."""
    n = d + 1
    nodes = st_nodes(d, M)
    L = len(nodes)
    monos = _monos(n, M)
    assert len(monos) == L == n_modes(M, n)
    # Vandermonde V[node][α] = node^α; Lagrange coefficients C = V⁻¹ (θ_l(node_k) = δ_kl)
    V = sp.Matrix(L, L, lambda i, j: sp.Rational(1))
    for i, x in enumerate(nodes):
        for j, a in enumerate(monos):
            v = Fraction(1)
            for xi, ai in zip(x, a):
                v *= xi ** ai
            V[i, j] = sp.Rational(v.numerator, v.denominator)
    Ci = V.inv()          # [α][l]
    C = [[Fraction(int(sp.fraction(Ci[a, l])[0]), int(sp.fraction(Ci[a, l])[1])) for l in range(L)]
         for a in range(L)]
    idx = {a: j for j, a in enumerate(monos)}

    def gram(shift_tau):
        G = [[Fraction(0)] * L for _ in range(L)]
        for i, a in enumerate(monos):
            for j, b in enumerate(monos):
                if shift_tau:
                    if b[-1] == 0:
                        continue
                    e = tuple(x + y for x, y in zip(a, b))
                    e = e[:-1] + (e[-1] - 1,)
                    G[i][j] = b[-1] * _prism_int(e)
                else:
                    G[i][j] = _prism_int(tuple(x + y for x, y in zip(a, b)))
        return G

    def cgc(G):  # Cᵀ G C
        out = [[Fraction(0)] * L for _ in range(L)]
        GC = [[sum(G[i][j] * C[j][l] for j in range(L)) for l in range(L)] for i in range(L)]
        for k in range(L):
            for l in range(L):
                out[k][l] = sum(C[i][k] * GC[i][l] for i in range(L))
        return out

    Mm = cgc(gram(False))
    Kt = cgc(gram(True))
    D = []
    for b in range(d):
        Db = [[Fraction(0)] * L for _ in range(L)]
        for l, x in enumerate(nodes):
            for m in range(L):
                s = Fraction(0)
                for j, a in enumerate(monos):
                    if a[b] == 0 or C[j][m] == 0:
                        continue
                    v = Fraction(a[b])
                    for c, (xc, ac) in enumerate(zip(x, a)):
                        v *= xc ** (ac - 1 if c == b else ac)
                    s += C[j][m] * v
                Db[l][m] = s
        D.append(Db)
    psis = dubiner_sympy(d, M)
    X = syms(d)
    Phi = np.array([[float(sp.N(p.subs({X[a]: sp.Rational(x[a].numerator, x[a].denominator) for a in range(d)}), 30))
                     for p in psis] for x in nodes])
    known = np.array([x[-1] == 0 for x in nodes])
    f = lambda A: np.array([[float(v) for v in row] for row in A])
    return dict(nodes=nodes, known=known, C=C, Kt_exact=Kt, M_exact=Mm, D_exact=D, Kt=f(Kt), Mm=f(Mm),
                D=np.array([f(Db) for Db in D]), Phi=Phi, monos=monos)


def euler_flux(q, d, gamma=GAMMA):
    """F_a(q) for conserved q [..., d+2] → [..., d, d+2]."""
    rho = q[..., 0]
    mom = q[..., 1:1 + d]
    E = q[..., 1 + d]
    u = mom / rho[..., None]
    p = (gamma - 1.0) * (E - 0.5 * np.sum(mom * u, axis=-1))
    F = np.zeros(q.shape[:-1] + (d, d + 2))
    for a in range(d):
        F[..., a, 0] = mom[..., a]
        for b in range(d):
            F[..., a, 1 + b] = mom[..., a] * u[..., b] + (p if a == b else 0.0)
        F[..., a, 1 + d] = u[..., a] * (E + p)
    return F, rho, p


def predict_cell(X, w, dt, M, gamma=GAMMA, tol=TOL, maxit=None):
    """Predictor of one cell.  X [d+1][d] vertices (x = X0 + J ξ);
    w [V = d+2][ℳ] reconstruction coefficients (Dubiner); dt the time step.

    Returns dict: q [𝓛][V] nodal space-time DOFs, iters, converged (bool),
    admissible (ρ > 0 and p > 0 at every node in every iterate)."""
    X = np.asarray(X, dtype=np.float64)
    d = X.shape[1]
    S = st_matrices(d, M)
    L = len(S["nodes"])
    known = S["known"]
    unk = ~known
    J = (X[1:] - X[0]).T                    # ∂x/∂ξ
    Jinv = np.linalg.inv(J)                 # ∂ξ/∂x: Jinv[b][a] = ∂ξ_b/∂x_a
    q = S["Phi"] @ np.asarray(w, dtype=np.float64).T      # [𝓛, V]: w(ξ_l) at every node
    q0 = q[known].copy()
    Kuu = S["Kt"][np.ix_(unk, unk)]
    Kuk = S["Kt"][np.ix_(unk, known)]
    Mu = S["Mm"][unk]
    scale = max(1.0, float(np.abs(q0).max()))
    maxit = maxit or MAXIT_FACTOR * (M + 1)
    admissible, converged, it = True, False, 0
    for it in range(1, maxit + 1):
        F, rho, p = euler_flux(q, d, gamma)                   # [𝓛, d, V]
        admissible &= bool(np.all(rho > 0) and np.all(p > 0))
        # Ĥ_l = Σ_m Σ_b D_b[l][m] Σ_a (∂ξ_b/∂x_a) F_a(q̂_m)
        H = np.zeros((L, d + 2))
        for b in range(d):
            Gb = np.einsum("a,mav->mv", Jinv[b], F)            # contravariant flux, direction b
            H += S["D"][b] @ Gb
        rhs = -dt * (Mu @ H) - Kuk @ q0
        qn = np.linalg.solve(Kuu, rhs)
        delta = float(np.abs(qn - q[unk]).max())
        q[unk] = qn
        if delta <= tol * scale:
            converged = True
            break
    if not converged and delta <= TOL_CAP * scale:
        converged = True
    F, rho, p = euler_flux(q, d, gamma)
    admissible &= bool(np.all(rho > 0) and np.all(p > 0))
    return dict(q=q, iters=it, converged=converged, admissible=admissible)


def eval_st(q, xi_tau, d, M):
    """Evaluate the space-time polynomial Σ_l θ_l(ξ̃) q̂_l at points ξ̃ [n][d+1]."""
    S = st_matrices(d, M)
    C = np.array([[float(v) for v in row] for row in S["C"]])   # [α][l]
    P = np.array([[np.prod([x ** e for x, e in zip(pt, a)]) for a in S["monos"]] for pt in xi_tau])  # [n][α]
    return P @ C @ q

"""Oracle: the CWENO reconstruction of one cell, literally.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  fp64 numpy, one cell at a
time, no fusion.  precompute_cell() builds one cell's stencil matrices from the
geometry and inverts them; apply_cell() is the reconstruction pass of
that cell; reconstruct_cell() does both on every call.

Steps (paper order):
 1. Stencils S_i^0 and S_i^s (oracle.mesh).
 2. Reconstruction matrix A[k][l] = (1/|T_j(k)|) ∫_{T_j(k)} ψ_l(ξ_i(x)) dx:
    the average over stencil cell j(k) of basis function l expressed in the
    OWNER's reference coordinates ξ_i (Eq. xietaTransf).
    Evaluated EXACTLY (up to fp64 rounding) by expanding ψ_l(t + C ξ') into
    monomials of the stencil cell's reference coordinate ξ' and using the
    Dirichlet formula avg_{T_E} ξ'^β = d! β! / (|β| + d)!  (no quadrature).
 3. P_opt (Eq. CWENO:Popt): constrained least squares.  The
    constraint row is the owner (k = 1): its averages are (ψ_1, 0, …, 0)
    because ∫_{T_E} ψ_l = 0 for l > 1 (orthogonality to the constant ψ_1,
    pinned in tests), so the constraint fixes p̂_1 = Q_i / ψ_1 and the rest
    minimises Σ_{k≥2} (Q_j(k) − A[k][1] p̂_1 − Σ_{l≥2} A[k][l] p̂_l)² —
    solved with the SVD pseudo-inverse of A[1:,1:] (numpy.linalg.pinv), which
    the Eulerian scheme may precompute once per cell.  (R10)
 4. P_s (Eq. CWENO:Ps): the (d+1)×(d+1) interpolation system on
    the sector cells, basis ψ_1..ψ_{d+1} (which span ℙ_1), numpy.linalg.solve.
 5. λ̄ = (λ_0, λ_s…)/Σ over VALID stencils, λ_0 = 1e5, λ_s = 1 (R5, R14).
 6. P_0 = (P_opt − Σ_s λ̄_s P_s)/λ̄_0  (Eq. CWENO:P0; sector vectors
    padded with zeros above mode d+1).
 7. σ_s = Σ_lm p̂^s_l p̂^s_m with the universal Σ; σ_0 from P_0 (R6).
 8. ω̃_s = λ̄_s / (σ_s + ε)^r, ω_s = ω̃_s / Σ_m ω̃_m, ε = 1e-14, r = 4
    (Eqs. weights/weights2), invalid sectors excluded (R14),
    per conserved variable (R7).
 9. w = Σ_{s=0}^{N_p} ω_s P_s  (Eq. CWENO:Prec, index read as s: R4).
"""
from __future__ import annotations

import math

import numpy as np

from .basis import basis_numeric, n_modes, psi1, sigma_numeric
from .mesh import OracleMesh

LAMBDA0 = 1e5
LAMBDAS = 1.0
EPS = 1e-14
R_EXP = 4


def monomial_average_table(d, M):
    """avg_{T_E} ξ^β = d! β! / (|β|+d)! on a dense (M+1)^d grid of exponents."""
    shape = (M + 1,) * d
    T = np.zeros(shape)
    for beta in np.ndindex(*shape):
        if sum(beta) <= M:
            num = math.factorial(d)
            for b in beta:
                num *= math.factorial(b)
            T[beta] = num / math.factorial(sum(beta) + d)
    return T


def affine_monomial_averages(t, C, exps, M):
    """For a batch of affine maps ξ = t + C ξ' ( t [B,d], C [B,d,d] ), return
    m [B, K] with m[:, k] = avg over T_E of Π_a (t_a + Σ_b C_ab ξ'_b)^{exps[k][a]}.

    Polynomials in ξ' are dense arrays [B, (M+1)^d]; each monomial of ξ is the
    product of the previous one with one linear form (exact expansion)."""
    B, d = t.shape
    shape = (B,) + (M + 1,) * d
    one = np.zeros(shape)
    one[(slice(None),) + (0,) * d] = 1.0
    polys = {(0,) * d: one}

    def times_linear(P, a):
        out = P * t[:, a].reshape((B,) + (1,) * d)
        for b in range(d):
            src = [slice(None)] + [slice(None)] * d
            dst = [slice(None)] + [slice(None)] * d
            src[1 + b] = slice(0, M)
            dst[1 + b] = slice(1, M + 1)
            out[tuple(dst)] += P[tuple(src)] * C[:, a, b].reshape((B,) + (1,) * d)
        return out

    for e in sorted((tuple(int(x) for x in e) for e in exps), key=sum):
        if e in polys:
            continue
        a = max(k for k in range(d) if e[k] > 0)
        prev = list(e)
        prev[a] -= 1
        polys[e] = times_linear(polys[tuple(prev)], a)
    T = monomial_average_table(d, M)
    m = np.empty((B, len(exps)))
    for k, e in enumerate(exps):
        m[:, k] = (polys[tuple(int(x) for x in e)] * T).reshape(B, -1).sum(axis=1)
    return m


def _affine(X):
    """x(ξ) = X0 + J ξ: returns X0 [d], J [d,d] (columns X_k − X_0)."""
    X0 = X[0]
    J = (X[1:] - X0).T
    return X0, J


def stencil_matrix(mesh: OracleMesh, i, cells_, M):
    """A[k][l] = average over (periodic image of) cell cells_[k] of ψ_l(ξ_i(x))."""
    d = mesh.d
    exps, Cb = basis_numeric(d, M)
    X0i, Ji = _affine(mesh.Xc(i))
    t = np.empty((len(cells_), d))
    C = np.empty((len(cells_), d, d))
    for k, j in enumerate(cells_):
        n = np.array(mesh.shift(i, j), dtype=np.float64)
        L = mesh.period if mesh.period is not None else np.zeros(d)
        Xj = mesh.Xc(j) + n * L
        X0j, Jj = _affine(Xj)
        t[k] = np.linalg.solve(Ji, X0j - X0i)
        C[k] = np.linalg.solve(Ji, Jj)
    m = affine_monomial_averages(t, C, exps, M)
    return m @ Cb.T   # [n, ℳ]


def precompute_cell(mesh: OracleMesh, i, M, central=None, sectors=None, valid=None):
    """The per-cell matrices of the Eulerian (fixed-mesh) scheme, built once
    ("precomputed, inverted and saved in the pre-processing stage"):

      A        [n_e, ℳ]   stencil matrix, row 0 = the cell itself
      pinv     [ℳ-1, n_e-1]  pseudo-inverse of A[1:,1:] (SVD, numpy.linalg.pinv):
               the minimiser of the reduced LSQ of P:136-149 (R10) is pinv·rhs
      As       [d+1][d+1, d+1]  the sector systems on ψ_1..ψ_{d+1},
               solved in the pass; None for an invalid sector (R14)
    plus the stencils themselves.  apply_cell() is the pass."""
    d = mesh.d
    if central is None:
        central = mesh.central_stencil(i)
    if sectors is None:
        sectors, valid = mesh.sector_stencils(i)
    A = stencil_matrix(mesh, i, central, M)                    # [n_e, ℳ]
    pinv = np.linalg.pinv(A[1:, 1:])                           # [ℳ-1, n_e-1]
    As = [stencil_matrix(mesh, i, sectors[s], M)[:, : d + 1] if valid[s] else None   # ψ_1..ψ_{d+1}
          for s in range(d + 1)]
    return dict(i=int(i), d=d, M=M, central=central, sectors=sectors, valid=valid, A=A, pinv=pinv, As=As,
                mesh=mesh if mesh.bc is not None else None)


def mesh_values(pre, Q, ids):
    """Q rows of the stencil cells; boundary ghosts (R37) through mesh.values."""
    if pre.get("mesh") is not None:
        return pre["mesh"].values(Q, ids)
    return Q[np.asarray(ids)]


def apply_cell(pre, Q, lam0=LAMBDA0, lams=LAMBDAS, eps=EPS, r=R_EXP):
    """One cell of the reconstruction pass with precompute_cell's matrices.

    Returns dict with w [V, ℳ] and the intermediates popt [V, ℳ], psec [d+1, V, d+1],
    P0 [V, ℳ], sigma [d+2, V], omega [d+2, V], lam [d+2] (normalised λ̄), valid [d+1]."""
    d, M, i = pre["d"], pre["M"], pre["i"]
    central, sectors, valid, A = pre["central"], pre["sectors"], pre["valid"], pre["A"]
    V = Q.shape[1]
    nm = n_modes(M, d)
    Sig = sigma_numeric(d, M)
    p1 = psi1(d)

    # --- P_opt: constrained LSQ
    Qs = mesh_values(pre, Q, central)                          # [n_e, V]
    popt = np.zeros((V, nm))
    popt[:, 0] = Q[i] / p1                                     # constraint row k=1
    rhs = Qs[1:] - np.outer(A[1:, 0], popt[:, 0])              # [n_e-1, V]
    popt[:, 1:] = (pre["pinv"] @ rhs).T                        # [ℳ-1, V] least-squares solution

    # --- sectorial P_s
    psec = np.zeros((d + 1, V, d + 1))
    for s in range(d + 1):
        if valid[s]:
            psec[s] = np.linalg.solve(pre["As"][s], mesh_values(pre, Q, sectors[s])).T

    # --- linear weights, normalised over valid stencils (R5, R14)
    lam = np.array([lam0] + [lams if valid[s] else 0.0 for s in range(d + 1)])
    lam = lam / lam.sum()

    # --- P_0
    P0 = popt.copy()
    for s in range(d + 1):
        P0[:, : d + 1] -= lam[s + 1] * psec[s]
    P0 /= lam[0]

    # --- oscillation indicators and weights
    cand = [P0] + [np.concatenate([psec[s], np.zeros((V, nm - d - 1))], axis=1) for s in range(d + 1)]
    sigma = np.array([np.einsum("vl,lm,vm->v", P, Sig, P) for P in cand])     # [d+2, V]
    wt = np.array([lam[s] / (sigma[s] + eps) ** r for s in range(d + 2)])     # [d+2, V]
    omega = wt / wt.sum(axis=0)
    w = sum(omega[s][:, None] * cand[s] for s in range(d + 2))
    return dict(w=w, popt=popt, psec=psec, P0=P0, sigma=sigma, omega=omega, lam=lam, valid=np.array(valid),
                central=central, sectors=sectors)


def reconstruct_cell(mesh: OracleMesh, i, Q, M, lam0=LAMBDA0, lams=LAMBDAS, eps=EPS, r=R_EXP,
                     central=None, sectors=None, valid=None):
    """Reconstruct cell i (SFC id).  Q: [N, V] cell averages in SFC order.
    = apply_cell(precompute_cell(...)): every call rebuilds the matrices."""
    pre = precompute_cell(mesh, i, M, central, sectors, valid)
    return apply_cell(pre, Q, lam0, lams, eps, r)


def reconstruct(mesh: OracleMesh, Q, M, cells_=None, **kw):
    """Coefficients [len(cells_), V, ℳ] for the given SFC cell ids (default: all)."""
    if cells_ is None:
        cells_ = range(mesh.N)
    out = []
    for i in cells_:
        out.append(reconstruct_cell(mesh, int(i), Q, M, **kw)["w"])
    return np.array(out)

"""Whole-operator pin of the oracle on C1 (BASELINE configs[0], 512 cells): the
same CWENO definition re-evaluated with 40 significant digits
(mpmath) and a DIFFERENT integration rule and LSQ method, against the oracle's
fp64 reconstruct_cell on every cell (SURVEY §8(c) "mpmath 40-digit
re-evaluation of C1").

Independent of the oracle's arithmetic: A is integrated with a collapsed
(Duffy) 3×3 Gauss-Legendre rule on T_E (exact for the degree-2 integrands of
M = 2) instead of the Dirichlet monomial formula; the constrained LSQ is solved
through the normal equations in 40-digit arithmetic instead of the SVD; the
basis and Σ come from their exact sympy forms (pinned in test_oracle_basis.py).
Only the integer stencils (pinned by the stencil invariants and the hand mesh)
are taken from the oracle.
"""
import numpy as np
import pytest
import sympy as sp

import gen
from oracle import basis as B
from oracle import reconstruct as R
from oracle.mesh import OracleMesh

mpmath = pytest.importorskip("mpmath")
mp = mpmath.mp


def _gl3():
    r = mp.sqrt(mp.mpf(3) / 5)
    x = [(1 - r) / 2, mp.mpf(1) / 2, (1 + r) / 2]
    w = [mp.mpf(5) / 18, mp.mpf(8) / 18, mp.mpf(5) / 18]
    return x, w


def _te_rule():
    """Duffy map (u, v) -> (u(1-v), v) of the unit square onto T_E, Jacobian (1-v)."""
    x, w = _gl3()
    pts, wts = [], []
    for a in range(3):
        for b in range(3):
            pts.append((x[a] * (1 - x[b]), x[b]))
            wts.append(w[a] * w[b] * (1 - x[b]))
    return pts, wts


def _mp_cell(m, i, Q, psis, Sig, rule, lam0=100000, lams=1, eps=mp.mpf("1e-14"), r=4):
    d = 2
    pts, wts = rule
    L = 1
    def verts(j, shift):
        return [[mp.mpf(float(m.X[j, k, a])) + shift[a] * L for a in range(d)] for k in range(d + 1)]
    Xi = verts(i, [0, 0])
    J = mp.matrix([[Xi[k + 1][a] - Xi[0][a] for k in range(d)] for a in range(d)])
    Ji = J ** -1
    def row(j, ncols):
        Xj = verts(j, m.shift(i, j))
        out = [mp.mpf(0)] * ncols
        for (u, v), wq in zip(pts, wts):
            x = [Xj[0][a] + u * (Xj[1][a] - Xj[0][a]) + v * (Xj[2][a] - Xj[0][a]) for a in range(d)]
            xi = Ji * mp.matrix([x[0] - Xi[0][0], x[1] - Xi[0][1]])
            for l in range(ncols):
                out[l] += 2 * wq * psis[l](xi[0], xi[1])          # average = ∫ / |T_E|
        return out
    central = m.central_stencil(i)
    sectors, valid = m.sector_stencils(i)
    nm = len(psis)
    V = Q.shape[1]
    A = [row(j, nm) for j in central]
    psi1 = mp.sqrt(2)
    p1 = [mp.mpf(float(Q[i, v])) / psi1 for v in range(V)]
    Ar = mp.matrix([[A[k][l] for l in range(1, nm)] for k in range(1, len(central))])
    AtA = Ar.T * Ar
    popt = []
    for v in range(V):
        rhs = mp.matrix([mp.mpf(float(Q[j, v])) - A[k][0] * p1[v] for k, j in enumerate(central) if k > 0])
        sol = mp.lu_solve(AtA, Ar.T * rhs)
        popt.append([p1[v]] + [sol[l] for l in range(nm - 1)])
    psec = []
    for s in range(d + 1):
        if not valid[s]:
            psec.append(None)
            continue
        As = mp.matrix([row(j, d + 1) for j in sectors[s]])
        psec.append([mp.lu_solve(As, mp.matrix([mp.mpf(float(Q[j, v])) for j in sectors[s]])) for v in range(V)])
    lam = [mp.mpf(lam0)] + [mp.mpf(lams) if valid[s] else mp.mpf(0) for s in range(d + 1)]
    tot = sum(lam)
    lam = [x / tot for x in lam]
    w = np.zeros((V, nm))
    for v in range(V):
        P0 = list(popt[v])
        for s in range(d + 1):
            if valid[s]:
                for l in range(d + 1):
                    P0[l] -= lam[s + 1] * psec[s][v][l]
        P0 = [x / lam[0] for x in P0]
        cands = [P0] + [[psec[s][v][l] if l <= d else mp.mpf(0) for l in range(nm)] if valid[s] else None
                        for s in range(d + 1)]
        wt = []
        for s, P in enumerate(cands):
            if P is None:
                wt.append(mp.mpf(0))
                continue
            sig = sum(P[a] * Sig[a, b] * P[b] for a in range(nm) for b in range(nm))
            wt.append(lam[s] / (sig + eps) ** r)
        tw = sum(wt)
        for l in range(nm):
            w[v, l] = float(sum(wt[s] / tw * cands[s][l] for s in range(d + 2) if cands[s] is not None))
    return w, central


def test_c1_whole_operator_40_digits():
    mp.dps = 40
    try:
        w_ = gen.make("C1")
        m = OracleMesh(w_["nodes"], w_["cells"], w_["period"], w_["M"])
        Q = w_["avgs"][m.perm]
        d, M = 2, 2
        psis = [sp.lambdify(B.syms(d), p, "mpmath") for p in B.dubiner_sympy(d, M)]
        S = B.sigma_sympy(d, M)
        Sig = mp.matrix([[mp.mpf(sp.N(S[a, b], 50)) for b in range(S.shape[1])] for a in range(S.shape[0])])
        rule = _te_rule()
        worst = 0.0
        for i in range(m.N):
            ref, central = _mp_cell(m, i, Q, psis, Sig, rule)
            got = R.reconstruct_cell(m, i, Q, M)["w"]
            s = np.abs(Q[np.asarray(central)]).max(axis=0)[:, None]      # R25 floor
            worst = max(worst, float((np.abs(got - ref) / np.maximum(np.abs(ref), s)).max()))
        print("C1 mpmath worst floored-relative error", worst)
        assert worst <= 1e-13, worst
    finally:
        mp.dps = 15

"""Oracle: face traces of the reconstruction polynomial.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The flux stage of the scheme (Eq. rusanov) evaluates the left and
right states at quadrature points of every face.  For a cell i (SFC id) and its
face f — the face opposite local vertex f of the orientation-fixed cell — the
face's d vertices are taken in ascending GLOBAL NODE ID order (a canonical
order both cells of the face agree on; reading, R31), the face rule is
the tensor Gauss rule with M+1 points per direction (Gauss–Legendre on an edge;
Gauss–Legendre × Gauss–Jacobi(1,0) collapsed onto a triangle), exact for degree
2M+1, with barycentric weights λ_q over those vertices; the physical point is
x_q = Σ_a λ_q[a] X_i[vertex_a] (cell i's unwrapped vertices) and the trace is the
blended polynomial at x_q:  w_i(x_q) = Σ_l w_l ψ_l(ξ_i(x_q)),  ξ_i = J_i⁻¹(x − X_0).

The rule comes from scipy's Gauss–Jacobi nodes (a library primitive); the basis
from the sympy monomial form (oracle.basis); the reference coordinate from a
linear solve with the cell's Jacobian — independent of the library, which
evaluates the basis at exact reference points Σ_a λ_a ξ(vertex_a) instead.
Pinned by tests/test_oracle_traces.py: rule exactness (Dirichlet formula on the
face simplex) and traces of reproduced polynomials equal the polynomial itself.
"""
from __future__ import annotations

import numpy as np
from scipy.special import roots_jacobi

from .basis import basis_numeric


def face_rule(d: int, M: int):
    """(lam [nq, d], weights [nq]) — barycentric weights over the face's d sorted
    vertices, weights summing to 1 (face average)."""
    n = M + 1
    x, wx = roots_jacobi(n, 0.0, 0.0)                 # Gauss–Legendre on [-1, 1]
    u, wu = (x + 1) / 2, wx / 2
    if d == 2:
        lam = np.stack([1 - u, u], axis=1)
        return lam, wu / wu.sum()
    y, wy = roots_jacobi(n, 1.0, 0.0)                 # weight (1 − y) on [-1, 1]
    v, wv = (y + 1) / 2, wy / 4
    pts, wts = [], []
    for a in range(n):
        for b in range(n):
            px, py = u[a] * (1 - v[b]), v[b]
            pts.append([1 - px - py, px, py])
            wts.append(wu[a] * wv[b])
    wts = np.array(wts)
    return np.array(pts), wts / wts.sum()


def face_vertices(mesh, i, f):
    """Local vertex indices of face f of cell i, sorted by global node id."""
    loc = [k for k in range(mesh.d + 1) if k != f]
    return sorted(loc, key=lambda k: mesh.cells[i][k])


def face_points(mesh, i, f, M):
    """Physical quadrature points [nq, d] of face f of cell i (cell i's unwrapped image)."""
    lam, _ = face_rule(mesh.d, M)
    V = mesh.X[i][face_vertices(mesh, i, f)]          # [d, d]
    return lam @ V


def eval_poly(mesh, i, w, x, M):
    """Cell i's polynomial with modal coefficients w [V, ℳ] at physical points x [n, d]."""
    exps, C = basis_numeric(mesh.d, M)
    X0 = mesh.X[i][0]
    J = (mesh.X[i][1:] - X0).T
    xi = np.linalg.solve(J, (x - X0).T).T             # [n, d]
    mono = np.prod(xi[:, None, :] ** exps[None, :, :], axis=2)   # [n, K]
    psi = mono @ C.T                                  # [n, ℳ]
    return psi @ w.T                                  # [n, V]


def cell_traces(mesh, i, w, M):
    """Traces [d+1, nq, V] of cell i's polynomial w [V, ℳ] on its faces."""
    return np.stack([eval_poly(mesh, i, w, face_points(mesh, i, f, M), M) for f in range(mesh.d + 1)])

"""GPU parity of the space-time predictor (cwreco_predict, NEXT-2)
against oracle/predictor.py, through the C-ABI.

The predictor consumes the reconstruction; both sides are given the SAME
coefficients (the GPU's cwreco_reconstruct output, itself checked against the
oracle elsewhere), so this isolates the predictor.  Tolerance: the library builds
its matrices by quadrature and a floating-point Vandermonde inverse and applies
K_uu⁻¹ pre-multiplied, the oracle uses exact rational matrices and solves every
iteration; κ(K_uu) ≤ 5e4 (3-D, M = 3) bounds the rounding difference, so
|q̂_gpu − q̂_orc| ≤ 1e-10 · max(1, max|q̂⁰|) per cell.  Node order: exact."""
import numpy as np
import pytest
import torch

import gen
import paper_1612_09335_b200 as P
from oracle import predictor as PR
from oracle.mesh import OracleMesh

pytestmark = pytest.mark.gpu


def _euler_state(x, d):
    r = 1.0 + 0.3 * np.sin(2 * np.pi * x[:, 0]) * np.cos(2 * np.pi * x[:, 1])
    vel = [0.4 * np.cos(2 * np.pi * x[:, 1]), -0.3 * np.sin(2 * np.pi * x[:, 0]), 0.2 + 0 * x[:, 0]][:d]
    p = 1.0 + 0.2 * np.cos(2 * np.pi * (x[:, 0] + x[:, d - 1]))
    return np.column_stack([r] + [r * v for v in vel] + [p / 0.4 + 0.5 * r * sum(v * v for v in vel)])


@pytest.mark.parametrize("d,n,M", [(2, 8, 1), (2, 8, 2), (2, 10, 3), (3, 3, 1), (3, 3, 2), (3, 3, 3)])
def test_predictor_parity(d, n, M):
    nodes, cells, period = gen.box_mesh(d, n, True, 0.15, 6)
    V = d + 2
    Q = gen.cell_averages(nodes, cells, period, lambda x: _euler_state(x, d), V)
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    m = OracleMesh(nodes, cells, period, M)
    Qs = torch.tensor(Q[m.perm], device="cuda")
    w = ctx.reconstruct(Qs)
    ctx.predictor_setup(1.4)
    onodes, nk = ctx.predictor_nodes()
    S = PR.st_matrices(d, M)
    assert nk == int(S["known"].sum())
    assert np.array_equal(onodes, np.array([[float(v) for v in x] for x in S["nodes"]]))
    h = 1.0 / n
    dt = 0.3 * h / (1.0 + np.sqrt(1.4 * 1.5 / 0.6))      # CFL ≈ 0.3 (|u| + c ≲ 2.6)
    iters = torch.empty(m.N, dtype=torch.int32, device="cuda")
    q = ctx.predict(w, dt, iters=iters).cpu().numpy()
    it = iters.cpu().numpy()
    wc = w.cpu().numpy()
    assert np.all(it > 0), it.min()
    worst, same_it = 0.0, 0
    cells_ = range(m.N) if m.N <= 400 else np.random.default_rng(0).choice(m.N, 400, replace=False)
    for i in cells_:
        r = PR.predict_cell(m.X[i], wc[i], dt, M)
        assert r["admissible"]
        assert (it[i] > 0) == r["converged"]
        scale = max(1.0, float(np.abs(r["q"][S["known"]]).max()))
        worst = max(worst, float(np.abs(q[i] - r["q"]).max()) / scale)
        same_it += int(it[i] == r["iters"])
    assert worst <= 1e-10, worst
    assert same_it >= 0.95 * len(cells_)
    # deterministic, and dt = 0 gives w at every node (constant in τ)
    q2 = ctx.predict(w, dt).cpu().numpy()
    assert np.array_equal(q, q2)
    # two CTAs walk every 32-cell group in turn (state carried across groups): same result
    ctx.set_option(P.OPT_MAX_CTAS, 2)
    assert np.array_equal(ctx.predict(w, dt).cpu().numpy(), q)
    ctx.set_option(P.OPT_MAX_CTAS, 0)
    # Δt = 0: H drops out and q_h(ξ, τ) = w(ξ) — q̂_l = w at the node's spatial point
    q0 = ctx.predict(w, 0.0).cpu().numpy()
    want = np.einsum("lm,cvm->clv", S["Phi"], wc)
    assert np.abs(q0 - want).max() <= 1e-10 * max(1.0, np.abs(want).max())   # κ(K_uu) ≤ 5e4
    # the τ = 0 rows (known DOFs) do not depend on Δt
    known = S["known"]
    assert np.array_equal(q[:, known], q0[:, known])


def test_predictor_contact_wave_on_gpu():
    """The exact-solution pin on the GPU path: contact wave (u, p constant, ρ a
    polynomial of degree M, given as exact Dubiner coefficients per cell) → the
    predictor reproduces ρ(x − u t) (and ρu, E) at every node of every cell."""
    import itertools
    import sympy as sp
    from oracle import basis as B
    d, n, M = 3, 3, 3
    nodes, cells, _ = gen.box_mesh(d, n, False, 0.1, 3)
    V = d + 2
    u = np.array([0.6, -0.35, 0.2])
    p0 = 1.1

    def state(x):
        r = 1.0 + 0.5 * x[:, 0] - 0.3 * x[:, 1] + 0.4 * x[:, 0] * x[:, 2] + 0.3 * x[:, 1] ** 3
        return np.column_stack([r] + [r * u[k] for k in range(d)] + [p0 / 0.4 + 0.5 * r * (u @ u)])
    ctx = P.Context(d, M, V, device=0)
    ctx.set_mesh(nodes, cells, None)
    ctx.build_stencils()
    ctx.predictor_setup(1.4)
    m = OracleMesh(nodes, cells, None, M)
    # orthonormal projection per cell with a 7^3-point collapsed Gauss rule (exact here)
    g, wg = np.polynomial.legendre.leggauss(7)
    g, wg = (g + 1) / 2, wg / 2
    pts, wts = [], []
    for a, b, c in itertools.product(range(7), repeat=3):
        pts.append((g[a] * (1 - g[b]) * (1 - g[c]), g[b] * (1 - g[c]), g[c]))
        wts.append(wg[a] * wg[b] * wg[c] * (1 - g[b]) * (1 - g[c]) ** 2)
    pts, wts = np.array(pts), np.array(wts)
    psi = np.array([np.broadcast_to(np.asarray(sp.lambdify(B.syms(d), p_, "numpy")(*pts.T), float), (len(pts),))
                    for p_ in B.dubiner_sympy(d, M)])
    W = np.empty((m.N, V, ctx.nm))
    for i in range(m.N):
        X = m.X[i]
        W[i] = ((psi * wts) @ state(X[0] + pts @ (X[1:] - X[0]))).T
    dt = 0.03
    q = ctx.predict(torch.tensor(W, device="cuda"), dt).cpu().numpy()
    onodes, _ = ctx.predictor_nodes()
    worst = 0.0
    for i in range(m.N):
        X = m.X[i]
        x = X[0] + onodes[:, :d] @ (X[1:] - X[0])
        exact = state(x - (onodes[:, d] * dt)[:, None] * u[None, :])
        worst = max(worst, np.abs(q[i] - exact).max() / np.abs(exact).max())
    assert worst < 1e-10, worst

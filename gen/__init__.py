"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module builds the meshes, initial conditions and cell averages of the five
workloads of BASELINE.json.  It holds NONE of the CWENO
method's arithmetic (no stencils, no basis, no least squares, no weights): it
only produces the *inputs* the method consumes, namely

  * ``nodes``  float64 [n_nodes, d]   vertex coordinates,
  * ``cells``  int64   [n_cells, d+1] simplex connectivity (input numbering),
  * ``period`` float64 [d] or None    periodic box lengths (None = open box),
  * ``avgs``   float64 [n_cells, V]   cell averages Q_i (PAPER.md:112-117,
                                       Eq. cellaverage) of the conserved vars.

Recipes (readings R20-R24, R28, R30 of SURVEY.md §8(c), restated in DESIGN.md):

  * 2D box: n x n squares, square (i, j) split along (i,j)->(i+1,j+1) into
    (v00, v10, v11) and (v00, v11, v01); cell id = 2*(j*n + i) + t.
  * 3D box: n^3 cubes, each split into 6 Kuhn tetrahedra along the main
    diagonal, one per axis permutation in ``itertools.permutations`` order;
    cell id = 6*((k*n + j)*n + i) + p.  Orientation is NOT fixed here (the
    method's ingest fixes it), so roughly half of the tetrahedra arrive
    negatively oriented.
  * Jitter: independent U(-a h, a h) per coordinate from
    ``numpy.random.default_rng(seed)``, drawn for every node in node-index
    order, then zeroed on nodes with any grid index equal to 0 (periodic box)
    or on the boundary (open box).
  * Averages: 2D by the 7-point degree-5 triangle rule, 3D by the collapsed
    (conical-product) Gauss-Jacobi rule with 3 points per direction (27
    points, degree 5).  Quadrature points are wrapped into the periodic box
    before the initial condition is evaluated.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

__all__ = [
    "CONFIGS", "box_mesh", "unwrap_cells", "ic_eval", "cell_averages", "make",
    "nvars_of", "polynomial_averages",
]

# name -> recipe.  n = cells per box edge.  C5's n is the per-N weak ladder
# (R26): 100/126/159/200 on 1/2/4/8 GPUs.
CONFIGS = {
    "C1": dict(d=2, n=16, M=2, ic="vortex", jitter=0.0, seed=0),
    "C2": dict(d=2, n=512, M=3, ic="vortex_jump", jitter=0.2, seed=2),
    "C3": dict(d=3, n=64, M=2, ic="explosion", jitter=0.0, seed=0),
    "C4": dict(d=3, n=128, M=3, ic="orszag_tang", jitter=0.1, seed=4),
    "C5": dict(d=3, n=100, M=3, ic="explosion", jitter=0.0, seed=0),
}
C5_WEAK_N = {1: 100, 2: 126, 4: 159, 8: 200}

_NVARS = {"vortex": 4, "vortex_jump": 4, "explosion": 5, "orszag_tang": 9}


def nvars_of(ic: str) -> int:
    return _NVARS[ic]


# --------------------------------------------------------------------------- mesh
def box_mesh(d: int, n: int, periodic: bool = True, jitter: float = 0.0,
             seed: int = 0):
    """Structured simplex mesh of the unit box (R28) with optional jitter (R30)."""
    if d not in (2, 3):
        raise ValueError("d must be 2 or 3")
    h = 1.0 / n
    m = n if periodic else n + 1  # nodes per edge
    idx = np.indices((m,) * d).reshape(d, -1)[::-1].T  # rows (i, j[, k]), i fastest
    nodes = idx.astype(np.float64) / n
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        J = rng.uniform(-jitter * h, jitter * h, size=nodes.shape)
        if periodic:
            fixed = np.any(idx == 0, axis=1)
        else:
            fixed = np.any((idx == 0) | (idx == n), axis=1)
        J[fixed] = 0.0
        nodes = nodes + J

    def nid(*ijk):
        ijk = [np.asarray(a) % m if periodic else np.asarray(a) for a in ijk]
        out = ijk[-1]
        for a in reversed(ijk[:-1]):
            out = out * m + a
        return out

    if d == 2:
        j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        i = i.ravel(); j = j.ravel()
        v00 = nid(i, j); v10 = nid(i + 1, j); v11 = nid(i + 1, j + 1); v01 = nid(i, j + 1)
        cells = np.empty((2 * n * n, 3), dtype=np.int64)
        cells[0::2] = np.stack([v00, v10, v11], axis=1)
        cells[1::2] = np.stack([v00, v11, v01], axis=1)
    else:
        k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        i = i.ravel(); j = j.ravel(); k = k.ravel()
        cells = np.empty((6 * n ** 3, 4), dtype=np.int64)
        for p, perm in enumerate(itertools.permutations(range(3))):
            off = np.zeros(3, dtype=np.int64)
            verts = [nid(i, j, k)]
            for ax in perm:
                off[ax] += 1
                verts.append(nid(i + off[0], j + off[1], k + off[2]))
            cells[p::6] = np.stack(verts, axis=1)
    period = np.ones(d) if periodic else None
    return nodes, cells, period


def unwrap_cells(nodes, cells, period):
    """Vertex coordinates per cell [n_cells, d+1, d], periodic images chosen by
    minimum image relative to the cell's first vertex (R16)."""
    X = nodes[cells]  # (N, d+1, d)
    if period is None:
        return X
    L = np.asarray(period, dtype=np.float64)
    X = X.copy()
    delta = X[:, 1:, :] - X[:, :1, :]
    X[:, 1:, :] -= np.where(delta > 0.5 * L, L, 0.0)
    X[:, 1:, :] += np.where(delta < -0.5 * L, L, 0.0)
    return X


# ------------------------------------------------------------------- quadrature
def _tri_rule7():
    """7-point degree-5 rule on the unit triangle; barycentric points, weights sum 1."""
    s15 = math.sqrt(15.0)
    a1 = (6.0 - s15) / 21.0
    a2 = (6.0 + s15) / 21.0
    w1 = (155.0 - s15) / 1200.0
    w2 = (155.0 + s15) / 1200.0
    bary = [(1 / 3, 1 / 3, 1 / 3)]
    w = [9.0 / 40.0]
    for a, wa in ((a1, w1), (a2, w2)):
        b = 1.0 - 2.0 * a
        bary += [(a, a, b), (a, b, a), (b, a, a)]
        w += [wa] * 3
    w = np.array(w)
    return np.array(bary), w / w.sum()


def _tet_rule27():
    """Conical-product Gauss-Jacobi rule (3 pts/direction) on the unit tet."""
    from scipy.special import roots_jacobi
    xu, wu = roots_jacobi(3, 0.0, 0.0)
    xv, wv = roots_jacobi(3, 1.0, 0.0)
    xw, ww = roots_jacobi(3, 2.0, 0.0)
    u = (xu + 1) / 2; v = (xv + 1) / 2; w = (xw + 1) / 2
    pts, wts = [], []
    for a in range(3):
        for b in range(3):
            for c in range(3):
                zeta = w[c]
                eta = v[b] * (1 - w[c])
                xi = u[a] * (1 - v[b]) * (1 - w[c])
                pts.append((1 - xi - eta - zeta, xi, eta, zeta))
                wts.append(wu[a] * wv[b] * ww[c])
    wts = np.array(wts)
    return np.array(pts), wts / wts.sum()


def _rule(d):
    return _tri_rule7() if d == 2 else _tet_rule27()


# ----------------------------------------------------------- initial conditions
def ic_eval(name: str, x: np.ndarray) -> np.ndarray:
    """Conserved variables at points x [P, d] (unit box coordinates)."""
    d = x.shape[1]
    if name in ("vortex", "vortex_jump"):
        # PAPER.md:565-576, Eqs. ShuVortIC/ShuVortDelta, evaluated at (10x, 10y) (R21)
        gam, eps = 1.4, 5.0
        X = 10.0 * x[:, 0] - 5.0
        Y = 10.0 * x[:, 1] - 5.0
        r2 = X * X + Y * Y
        e = np.exp(0.5 * (1.0 - r2))
        u = 1.0 - eps / (2 * np.pi) * e * Y
        v = 1.0 + eps / (2 * np.pi) * e * X
        dT = -(gam - 1.0) * eps ** 2 / (8 * gam * np.pi ** 2) * np.exp(1.0 - r2)
        rho = (1.0 + dT) ** (1.0 / (gam - 1.0))
        p = (1.0 + dT) ** (gam / (gam - 1.0))
        if name == "vortex_jump":  # R22
            rr = np.sqrt((x[:, 0] - 0.5) ** 2 + (x[:, 1] - 0.5) ** 2)
            f = np.where(rr < 0.25, 10.0, 1.0)
            rho = rho * f
            p = p * f
        E = p / (gam - 1.0) + 0.5 * rho * (u * u + v * v)
        return np.stack([rho, rho * u, rho * v, E], axis=1)
    if name == "explosion":
        # Sod states, R23: ball r < 0.4 centred in the unit cube
        gam = 1.4
        c = 0.5
        rr = np.sqrt(((x - c) ** 2).sum(axis=1))
        inside = rr < 0.4
        rho = np.where(inside, 1.0, 0.125)
        p = np.where(inside, 1.0, 0.1)
        z = np.zeros_like(rho)
        mom = [z] * 3 if d == 3 else [z] * 2
        return np.stack([rho, *mom, p / (gam - 1.0)], axis=1)
    if name == "orszag_tang":
        # PAPER.md:884 Eq. Orszag-Tang-IC at (2 pi x, 2 pi y), z-independent (R24)
        gam = 5.0 / 3.0
        X = 2 * np.pi * x[:, 0]
        Y = 2 * np.pi * x[:, 1]
        rho = np.full_like(X, gam * gam)
        u = -np.sin(Y); v = np.sin(X); w = np.zeros_like(X)
        p = np.full_like(X, gam)
        s4p = math.sqrt(4 * np.pi)
        Bx = -s4p * np.sin(Y); By = s4p * np.sin(2 * X); Bz = np.zeros_like(X)
        psi = np.zeros_like(X)
        E = p / (gam - 1.0) + 0.5 * rho * (u * u + v * v + w * w) + (Bx * Bx + By * By + Bz * Bz) / (8 * np.pi)
        return np.stack([rho, rho * u, rho * v, rho * w, E, Bx, By, Bz, psi], axis=1)
    raise ValueError(f"unknown initial condition {name!r}")


def cell_averages(nodes, cells, period, func, nvars: int, chunk: int = 1 << 16):
    """Quadrature cell averages of ``func(points [P,d]) -> [P, nvars]``.

    Chunks are independent (same operations per cell whatever the chunking), so
    they are evaluated on a thread pool (numpy releases the GIL)."""
    import concurrent.futures as cf
    import os
    d = nodes.shape[1]
    bary, w = _rule(d)
    out = np.empty((cells.shape[0], nvars), dtype=np.float64)

    def work(s):
        X = unwrap_cells(nodes, cells[s:s + chunk], period)  # (c, d+1, d)
        pts = np.einsum("qk,ckd->cqd", bary, X)  # (c, q, d)
        P = pts.reshape(-1, d)
        if period is not None:
            P = P - np.floor(P / period) * period
        vals = func(P).reshape(pts.shape[0], pts.shape[1], nvars)
        out[s:s + chunk] = np.einsum("q,cqv->cv", w, vals)

    starts = range(0, cells.shape[0], chunk)
    nw = min(32, os.cpu_count() or 1)
    if len(starts) == 1 or nw == 1:
        for s in starts:
            work(s)
    else:
        with cf.ThreadPoolExecutor(nw) as ex:
            list(ex.map(work, starts))
    return out


def polynomial_averages(nodes, cells, coeffs_by_var):
    """Exact-to-rounding averages of global polynomials of degree <= 5 on an OPEN
    mesh (used by the polynomial-reproduction pins).  ``coeffs_by_var`` is a list
    of callables f(points [P,d]) -> [P]."""
    def f(P):
        return np.stack([g(P) for g in coeffs_by_var], axis=1)
    return cell_averages(nodes, cells, None, f, len(coeffs_by_var))


def make(name: str, n: int | None = None):
    """Build workload ``name`` (C1..C5); ``n`` overrides the box resolution."""
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    nodes, cells, period = box_mesh(cfg["d"], cfg["n"], True, cfg["jitter"], cfg["seed"])
    V = nvars_of(cfg["ic"])
    ic = cfg["ic"]
    avgs = cell_averages(nodes, cells, period, lambda P: ic_eval(ic, P), V)
    return dict(name=name, d=cfg["d"], M=cfg["M"], V=V, n=cfg["n"], ic=ic,
                nodes=nodes, cells=cells, period=period, avgs=avgs)

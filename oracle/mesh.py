"""Oracle: mesh geometry, space-filling-curve order, adjacency and CWENO stencils.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy for whole-mesh
arrays, pure Python + ``fractions.Fraction`` (exact rational arithmetic) for
every geometric decision that selects a stencil cell.

Paper passages followed:
  * affine map / vertices of T_i ............ P:94-102 (Eq. xietaTransf)
  * central stencil S_i^0, n_e = d·ℳ cells,
    j(1) = i, "recursively adding neighbors
    of elements that have been already
    selected" .............................. P:129-134 (Eq. stencil)
  * sectorial stencils: d+1 stencils of d+1
    cells, same recursion, "selecting only
    those elements whose barycenter lies in
    the open cone defined by one vertex and
    the opposite face" ..................... P:156
  * Neumann (face) neighbours ............... P:452;  Voronoi (node) nbrs P:351

Readings: R11 face neighbours drive the recursion, node neighbours
only as the sector fallback; R12 layer order by (exact squared barycentre
distance, SFC id), last layer truncated; R13 open cone of owner vertex v =
{x : λ_w(x) > 0 for all w ≠ v} in the owner's barycentric coordinates, decided
exactly; R14 sector fallback / invalid sectors; R16 periodic minimum image;
R28 orientation fix; R29 IEEE-specified barycentres and Morton keys.

Exactness: every cone test, distance comparison and orientation sign is
evaluated on the *given* doubles (unwrapped vertex coordinates) with exact
rational arithmetic, so the decision is the geometric truth for those doubles.
Only two steps are specified as IEEE double operations (and are therefore
reproducible bit-for-bit by any implementation doing the same operations):
the barycentre b = ((X0+X1)+X2[+X3])/(d+1) used for the periodic image choice
and the Morton key.  STENCIL PARITY IS UNPINNED against the paper (figures
stripped): pinned by invariants only.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from .basis import n_modes

__all__ = ["OracleMesh", "StencilExhausted", "MeshError"]


class StencilExhausted(RuntimeError):
    pass


class MeshError(ValueError):
    pass


def _orient_frac(pts):
    """Exact orientation determinant of d+1 points (Fractions) in R^d."""
    d = len(pts) - 1
    p0 = pts[0]
    rows = [[pts[k][a] - p0[a] for a in range(d)] for k in range(1, d + 1)]
    if d == 2:
        return rows[0][0] * rows[1][1] - rows[0][1] * rows[1][0]
    (a, b, c), (e, f, g), (h, i, j) = rows
    return a * (f * j - g * i) - b * (e * j - g * h) + c * (e * i - f * h)


def _sign(x):
    return (x > 0) - (x < 0)


class OracleMesh:
    """Whole-mesh arrays in SFC order + per-cell exact stencil construction.

    Attributes (SFC numbering, i.e. after the Morton permutation):
      perm    [N]        perm[s] = input id of SFC cell s
      cells   [N, d+1]   node ids after the orientation fix
      X       [N, d+1, d] unwrapped vertex coordinates (doubles)
      bary    [N, d]     IEEE barycentres ((X0+X1)+X2[+X3])/(d+1)
      nbr     [N, d+1]   face neighbour across the face opposite local vertex f (-1: none)
      node_cells CSR     (nc_ptr, nc_idx) node -> sorted SFC cell ids
    """

    def __init__(self, nodes, cells, period, M, bc=None, mom0=None):
        """bc: None, or per side s = 2·axis + (0 low, 1 high) of the nodes' bounding
        box: 0 none, 1 transmissive, 2 wall — boundary ghost cells by reflection
        (R37, open meshes only); mom0: index of ρu_1 in the conserved vector (wall)."""
        nodes = np.asarray(nodes, dtype=np.float64)
        cells = np.asarray(cells, dtype=np.int64)
        self.d = d = nodes.shape[1]
        if d not in (2, 3) or cells.shape[1] != d + 1:
            raise MeshError("bad shapes")
        self.M = M
        self.n_e = d * n_modes(M, d)
        self.period = None if period is None else np.asarray(period, dtype=np.float64)
        if cells.min() < 0 or cells.max() >= nodes.shape[0]:
            raise MeshError("cell references a missing node")
        for a in range(d + 1):
            for b in range(a + 1, d + 1):
                if np.any(cells[:, a] == cells[:, b]):
                    raise MeshError("cell with repeated vertex")
        X = self._unwrap(nodes, cells)
        cells, X = self._orient(cells, X)
        bary = self._bary(X)
        perm = self._morton_perm(bary, nodes)
        self.perm = perm
        self.cells = cells[perm]
        self.X = X[perm]
        self.bary = bary[perm]
        self.N = self.cells.shape[0]
        self.n_nodes = nodes.shape[0]
        self._adjacency()
        self._frac_cache = {}
        self.bc = None
        if bc is not None:
            if self.period is not None:
                raise MeshError("boundary ghost cells need an open mesh")
            if len(bc) != 2 * d:
                raise MeshError("bc needs one entry per box side")
            self.bc = [int(x) for x in bc]
            self.mom0 = mom0
            lo, hi = nodes.min(axis=0), nodes.max(axis=0)
            self.plane = [float(lo[s // 2]) if s % 2 == 0 else float(hi[s // 2]) for s in range(2 * d)]
            self._gX = {}

    # ------------------------------------------------- boundary ghosts (R37)
    # Ghost id N + s·N + k = the mirror image of real cell k across box side s
    # (x_a = c, a = s // 2): vertices X'_a = c + (c − X_a) in IEEE double, the last
    # two swapped (orientation, R28).  Face adjacency: a real boundary face on an
    # active side s borders the mirror of its own cell; a ghost's faces border the
    # mirrors (same side) of its source's neighbours, its mirrored face on s borders
    # the source itself, and faces on other sides border nothing (no double
    # reflection).  Node (Voronoi) neighbours — the R14 fallback — stay real cells.
    def is_ghost(self, j):
        return j >= self.N

    def ghost_of(self, j):
        """(side s, source k) of ghost id j."""
        s, k = divmod(j - self.N, self.N)
        return s, k

    def face_side(self, k, f):
        """Active box side containing face f of real cell k (all its vertices on the
        plane, exactly), or -1."""
        if self.bc is None:
            return -1
        d = self.d
        V = [self.X[k, v] for v in range(d + 1) if v != f]
        for s in range(2 * d):
            if self.bc[s] and all(x[s // 2] == self.plane[s] for x in V):
                return s
        return -1

    def Xc(self, j):
        """Vertex coordinates [d+1][d] of real or ghost cell j."""
        if j < self.N:
            return self.X[j]
        g = self._gX.get(j)
        if g is None:
            s, k = self.ghost_of(j)
            a, c = s // 2, self.plane[s]
            g = self.X[k].copy()
            g[:, a] = c + (c - self.X[k][:, a])
            g[[self.d - 1, self.d]] = g[[self.d, self.d - 1]]
            self._gX[j] = g
        return g

    def neighbours(self, c):
        """Face neighbours of real or ghost cell c (ghosts included when bc is set)."""
        if c < self.N:
            out = []
            for f in range(self.d + 1):
                nb = int(self.nbr[c, f])
                if nb >= 0:
                    out.append(nb)
                else:
                    s = self.face_side(c, f)
                    if s >= 0:
                        out.append(self.N + s * self.N + c)
            return out
        s, k = self.ghost_of(c)
        out = []
        for f in range(self.d + 1):
            nb = int(self.nbr[k, f])
            if nb >= 0:
                out.append(self.N + s * self.N + nb)
            elif self.face_side(k, f) == s:
                out.append(k)
        return out

    def values(self, Q, ids):
        """Averages of real or ghost cells: a ghost carries its source's averages,
        with the momentum component normal to a WALL side negated (R37)."""
        ids = [int(j) for j in ids]
        out = np.empty((len(ids), Q.shape[1]))
        for r, j in enumerate(ids):
            if j < self.N:
                out[r] = Q[j]
            else:
                s, k = self.ghost_of(j)
                out[r] = Q[k]
                if self.bc[s] == 2 and self.mom0 is not None:
                    out[r, self.mom0 + s // 2] = -Q[k, self.mom0 + s // 2]
        return out

    # -------------------------------------------------------------- geometry
    def _unwrap(self, nodes, cells):
        """R16: minimum image of each vertex relative to the cell's first vertex."""
        X = nodes[cells].copy()
        if self.period is None:
            return X
        L = self.period
        delta = X[:, 1:, :] - X[:, :1, :]
        hi = delta > 0.5 * L
        lo = delta < -0.5 * L
        Xs = X[:, 1:, :]
        Xs = np.where(hi, Xs - L, np.where(lo, Xs + L, Xs))
        X[:, 1:, :] = Xs
        return X

    def _orient(self, cells, X):
        """R28: make every cell positively oriented (exact sign); swap last two vertices."""
        d = self.d
        E = X[:, 1:, :] - X[:, :1, :]
        if d == 2:
            t1 = E[:, 0, 0] * E[:, 1, 1]
            t2 = E[:, 0, 1] * E[:, 1, 0]
            det = t1 - t2
            perm_sum = np.abs(t1) + np.abs(t2)
        else:
            a, b, c = E[:, 0, 0], E[:, 0, 1], E[:, 0, 2]
            e, f, g = E[:, 1, 0], E[:, 1, 1], E[:, 1, 2]
            h, i, j = E[:, 2, 0], E[:, 2, 1], E[:, 2, 2]
            det = a * (f * j - g * i) - b * (e * j - g * h) + c * (e * i - f * h)
            perm_sum = (np.abs(a) * (np.abs(f * j) + np.abs(g * i)) + np.abs(b) * (np.abs(e * j) + np.abs(g * h))
                        + np.abs(c) * (np.abs(e * i) + np.abs(f * h)))
        sign = np.sign(det).astype(np.int64)
        unsure = np.abs(det) <= 1e-10 * perm_sum
        for c in np.nonzero(unsure)[0]:
            pts = [[Fraction(float(v)) for v in X[c, k]] for k in range(d + 1)]
            sign[c] = _sign(_orient_frac(pts))
        if np.any(sign == 0):
            raise MeshError("zero-volume cell")
        neg = sign < 0
        cells = cells.copy()
        X = X.copy()
        cells[neg, d - 1], cells[neg, d] = cells[neg, d].copy(), cells[neg, d - 1].copy()
        tmp = X[neg, d - 1, :].copy()
        X[neg, d - 1, :] = X[neg, d, :]
        X[neg, d, :] = tmp
        return cells, X

    def _bary(self, X):
        """R29: b = ((X0+X1)+X2[+X3])/(d+1), IEEE double, left to right."""
        s = X[:, 0, :] + X[:, 1, :]
        s = s + X[:, 2, :]
        if self.d == 3:
            s = s + X[:, 3, :]
        return s / float(self.d + 1)

    def _morton_perm(self, bary, nodes):
        """R29: Morton key of the wrapped barycentre; stable sort by (key, input id)."""
        d = self.d
        k = 31 if d == 2 else 21
        if self.period is not None:
            u = bary / self.period
            u = u - np.floor(u)
        else:
            lo = nodes.min(axis=0)
            hi = nodes.max(axis=0)
            u = (bary - lo) / (hi - lo)
        q = np.floor(u * float(1 << k))
        q = np.clip(q, 0, (1 << k) - 1).astype(np.uint64)
        key = np.zeros(bary.shape[0], dtype=np.uint64)
        for t in range(k):
            for a in range(d):
                bit = (q[:, a] >> np.uint64(t)) & np.uint64(1)
                key |= bit << np.uint64(d * t + a)
        ids = np.arange(bary.shape[0], dtype=np.int64)
        return np.lexsort((ids, key))

    # -------------------------------------------------------------- topology
    def _adjacency(self):
        d = self.d
        N = self.N
        faces = []
        for f in range(d + 1):
            cols = [k for k in range(d + 1) if k != f]
            faces.append(np.sort(self.cells[:, cols], axis=1))
        F = np.concatenate(faces, axis=0)                  # (N*(d+1), d)
        owner = np.tile(np.arange(N, dtype=np.int64), d + 1)
        lface = np.repeat(np.arange(d + 1, dtype=np.int64), N)
        order = np.lexsort(tuple(F[:, a] for a in range(d - 1, -1, -1)))
        Fs = F[order]
        same = np.all(Fs[1:] == Fs[:-1], axis=1)
        if np.any(same[1:] & same[:-1]):
            raise MeshError("non-manifold face (shared by > 2 cells)")
        nbr = -np.ones((N, d + 1), dtype=np.int64)
        idx = np.nonzero(same)[0]
        a = order[idx]
        b = order[idx + 1]
        if np.any(owner[a] == owner[b]):
            raise MeshError("degenerate cell")
        nbr[owner[a], lface[a]] = owner[b]
        nbr[owner[b], lface[b]] = owner[a]
        # duplicate cells: two cells sharing all d+1 faces
        self.nbr = nbr
        srt = np.sort(self.cells, axis=1)
        o2 = np.lexsort(tuple(srt[:, a] for a in range(d, -1, -1)))
        if np.any(np.all(srt[o2][1:] == srt[o2][:-1], axis=1)):
            raise MeshError("duplicate cell")
        flat = self.cells.ravel()
        cell_of = np.repeat(np.arange(N, dtype=np.int64), d + 1)
        o = np.lexsort((cell_of, flat))
        self.nc_idx = cell_of[o]
        counts = np.bincount(flat, minlength=self.n_nodes)
        self.nc_ptr = np.concatenate([[0], np.cumsum(counts)])

    # ------------------------------------------------- exact per-cell helpers
    def _fr(self, c):
        """Exact vertex coordinates and vertex sums S_c of cell c (Fractions)."""
        got = self._frac_cache.get(c)
        if got is None:
            Xc = self.Xc(c)
            Xf = [[Fraction(float(v)) for v in Xc[k]] for k in range(self.d + 1)]
            S = [sum(Xf[k][a] for k in range(self.d + 1)) for a in range(self.d)]
            got = (Xf, S)
            if len(self._frac_cache) > 200000:
                self._frac_cache.clear()
            self._frac_cache[c] = got
        return got

    def shift(self, i, j):
        """Periodic image of cell j nearest to cell i (R16): integer shift n with
        the IEEE recipe r = b_j - b_i; while r > L/2: r -= L, n -= 1; while r < -L/2: r += L, n += 1."""
        n = [0] * self.d
        if self.period is None:
            return n
        for a in range(self.d):
            L = float(self.period[a])
            r = float(self.bary[j, a]) - float(self.bary[i, a])
            while r > 0.5 * L:
                r -= L
                n[a] -= 1
            while r < -0.5 * L:
                r += L
                n[a] += 1
        return n

    def disp(self, i, j):
        """Exact (d+1)·(barycentre_j' − barycentre_i), j' the image of j near i."""
        d = self.d
        _, Si = self._fr(i)
        _, Sj = self._fr(j)
        n = self.shift(i, j)
        out = []
        for a in range(d):
            L = Fraction(float(self.period[a])) if self.period is not None else Fraction(0)
            out.append(Sj[a] - Si[a] + (d + 1) * n[a] * L)
        return out

    def key(self, i, j):
        D = self.disp(i, j)
        return (sum(x * x for x in D), j)

    def lambda_signs(self, i, j):
        """Exact signs of the owner's barycentric coordinates λ_w of the barycentre
        of (the periodic image of) cell j, w = 0..d."""
        d = self.d
        Xf, Si = self._fr(i)
        W = [[(d + 1) * Xf[k][a] - Si[a] for a in range(d)] for k in range(d + 1)]
        D = self.disp(i, j)
        signs = []
        for w in range(d + 1):
            pts = [D if k == w else W[k] for k in range(d + 1)]
            signs.append(_sign(_orient_frac(pts)))
        return signs

    def in_cone(self, i, j, v):
        """R13: open cone of owner vertex v (apex v, through the opposite face)."""
        s = self.lambda_signs(i, j)
        return all(s[w] > 0 for w in range(self.d + 1) if w != v)

    # ---------------------------------------------------------------- stencils
    def central_stencil(self, i):
        """S_i^0 (R11-R12): layered face-neighbour BFS from i; each new
        layer sorted by (exact squared distance, SFC id); last layer truncated."""
        n_e = self.n_e
        S = [i]
        inS = {i}
        frontier = [i]
        while len(S) < n_e:
            cand = set()
            for c in frontier:
                for nb in self.neighbours(c):
                    if nb not in inS:
                        cand.add(nb)
            if not cand:
                raise StencilExhausted(f"central stencil of cell {i} exhausted at {len(S)} < {n_e}")
            order = sorted(cand, key=lambda j: self.key(i, j))
            take = order[: n_e - len(S)]
            S += take
            inS.update(take)
            frontier = take
        return S

    def node_neighbours(self, cells_):
        out = set()
        for c in cells_:
            if c >= self.N:
                continue            # ghosts contribute no node neighbours (R37)
            for nd in self.cells[c]:
                out.update(int(x) for x in self.nc_idx[self.nc_ptr[nd]:self.nc_ptr[nd + 1]])
        return out

    def sector_stencil(self, i, v):
        """S_i^s for owner vertex v (R13-R14).  Returns (cells, valid)."""
        d = self.d
        S = [i]
        seen = {i}
        frontier = [i]
        while len(S) < d + 1:
            cand = set()
            for c in frontier:
                for nb in self.neighbours(c):
                    if nb not in seen:
                        cand.add(nb)
            seen.update(cand)
            acc = [j for j in cand if self.in_cone(i, j, v)]
            if not acc:
                cand2 = self.node_neighbours(S) - set(S)
                acc = [j for j in cand2 if self.in_cone(i, j, v)]
                if not acc:
                    return S, False
            acc.sort(key=lambda j: self.key(i, j))
            take = acc[: d + 1 - len(S)]
            S += take
            seen.update(take)
            frontier = take
        # non-degenerate iff the d+1 barycentres are affinely independent (exact)
        pts = [[Fraction(0)] * d] + [self.disp(i, j) for j in S[1:]]
        return S, _orient_frac(pts) != 0

    def sector_stencils(self, i):
        out, valid = [], []
        for v in range(self.d + 1):
            S, ok = self.sector_stencil(i, v)
            out.append(S + [-1] * (self.d + 1 - len(S)))
            valid.append(bool(ok))
        return out, valid

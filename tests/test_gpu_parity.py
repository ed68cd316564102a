"""GPU parity of the CUDA reconstruction (through the C-ABI) against the CPU oracle.

Tolerance (north_star: 1e-11 relative, fp64; reading R25): for every output
coefficient, |c_gpu − c_oracle| ≤ 1e-11 · max(|c_oracle|, s_{i,v}) with
s_{i,v} = max over the central stencil of |Q_{j,v}|; a variable that is
identically zero on the stencil (s = 0) must come out exactly 0.
Stencils and SFC order: bit-exact.  Both CUDA kernels: bitwise identical.
"""
import numpy as np
import pytest
import torch

import gen
import paper_1612_09335_b200 as P
from oracle import reconstruct as R
from oracle.mesh import OracleMesh

pytestmark = pytest.mark.gpu
TOL = 1e-11


def floored_err(got, ref, Q, central):
    """max floored-relative error of one cell: got/ref [V, ℳ], Q global [N, V]."""
    s = np.abs(Q[np.asarray(central)]).max(axis=0)[:, None]           # [V, 1]
    zero = (s == 0)[:, 0]
    if np.any(zero):
        assert np.all(got[zero] == 0.0)
    den = np.maximum(np.abs(ref), s)
    e = np.abs(got - ref)
    e = np.where(den > 0, e / np.where(den > 0, den, 1), e)
    return float(e.max())


def _run(ctx, Q, kernel):
    ctx.set_kernel(kernel)
    out = ctx.reconstruct(torch.tensor(Q, device="cuda"))
    torch.cuda.synchronize()
    return out.cpu().numpy()


CASES = [
    # name, d, n, M, jitter, periodic, V, n_check (None = all cells)
    ("2d-M2", 2, 16, 2, 0.0, True, 4, None),
    ("2d-M3-jit", 2, 24, 3, 0.2, True, 4, None),
    ("2d-M1", 2, 12, 1, 0.1, True, 2, None),
    ("2d-M4-jit", 2, 14, 4, 0.1, True, 3, 150),
    ("2d-M2-open", 2, 11, 2, 0.15, False, 3, None),        # boundary cells: invalid sectors, extras
    ("3d-M2", 3, 6, 2, 0.0, True, 5, 250),
    ("3d-M3-jit", 3, 6, 3, 0.1, True, 9, 150),
    ("3d-M1-open", 3, 5, 1, 0.1, False, 1, None),
    ("3d-M2-open", 3, 5, 2, 0.1, False, 5, 200),
]


@pytest.mark.parametrize("family", ["0", "1"], ids=["cellvar", "rowblk"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_small_mesh_parity(case, family):
    """Both kernel families (CWRECO_OPT_FAMILY: 0 = one thread per (cell, variable),
    1 = row-block where instantiated, ℳ ≥ 10) against the oracle and k_simple."""
    name, d, n, M, jit, per, V, ncheck = case
    nodes, cells, period = gen.box_mesh(d, n, per, jit, 21)
    rng = np.random.default_rng(3)
    Qin = rng.standard_normal((cells.shape[0], V)) * 2.0 + 3.0
    ctx = P.setup_context(nodes, cells, period, M, V, device=0, family=int(family))
    m = OracleMesh(nodes, cells, period, M)
    assert np.array_equal(ctx.permutation(), m.perm)
    Q = Qin[m.perm]
    a = _run(ctx, Q, "pipelined")
    b = _run(ctx, Q, "simple")
    assert np.array_equal(a, b), "kernels differ"
    assert np.all(np.isfinite(a))
    sel = range(m.N) if ncheck is None else rng.choice(m.N, ncheck, replace=False)
    worst = 0.0
    for i in sel:
        r = R.reconstruct_cell(m, int(i), Q, M)
        worst = max(worst, floored_err(a[i], r["w"], Q, r["central"]))
    assert worst <= TOL, (name, worst)
    # conservation of the cell average (R17): w[0]·ψ1 = Q_i
    psi1 = np.sqrt(2.0 if d == 2 else 6.0)
    assert np.abs(a[:, :, 0] * psi1 - Q).max() <= 4e-16 * np.abs(Q).max()


def test_debug_tap_intermediates():
    nodes, cells, period = gen.box_mesh(2, 12, False, 0.15, 2)
    V, M = 3, 2
    Qin = np.random.default_rng(0).standard_normal((cells.shape[0], V))
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    m = OracleMesh(nodes, cells, period, M)
    Q = Qin[m.perm]
    sel = np.arange(0, m.N, 3)
    dbg = ctx.reconstruct_debug(torch.tensor(Q, device="cuda"), sel)
    full = _run(ctx, Q, "pipelined")
    assert np.array_equal(dbg["w"], full[sel])
    for q, i in enumerate(sel):
        r = R.reconstruct_cell(m, int(i), Q, M)
        s = np.abs(Q[r["central"]]).max()
        assert np.abs(dbg["popt"][q] - r["popt"]).max() <= 1e-12 * s
        assert np.abs(dbg["psec"][q] - r["psec"]).max() <= 1e-12 * s
        assert np.abs(dbg["sigma"][q] - r["sigma"]).max() <= 1e-9 * np.abs(r["sigma"]).max() + 1e-20 * s * s
        assert np.abs(dbg["omega"][q] - r["omega"]).max() <= 1e-7
        assert np.abs(dbg["omega"][q].sum(axis=0) - 1.0).max() <= 1e-14       # Σω = 1


def test_constant_and_linear_data():
    # constant data: σ = 0, ω = λ̄, w = (Q/ψ1, 0, …) exactly;  linear data: w exact (ℙ1)
    nodes, cells, _ = gen.box_mesh(3, 6, False, 0.1, 4)
    ctx = P.setup_context(nodes, cells, None, 2, 2, device=0)
    perm = ctx.permutation()
    X = nodes[cells].mean(axis=1)
    Qc = np.full((cells.shape[0], 2), 1.25)
    w = _run(ctx, Qc[perm], "pipelined")
    assert np.all(w[:, :, 1:] == 0.0) and np.all(w[:, :, 0] == 1.25 / np.sqrt(6.0))
    lin = 0.3 + X @ np.array([1.0, -2.0, 0.5])                 # average of a linear field = value at barycentre
    Ql = np.stack([lin, -lin], axis=1)[perm]
    w = _run(ctx, Ql, "pipelined")
    m = OracleMesh(nodes, cells, None, 2)
    for i in range(0, m.N, 37):
        r = R.reconstruct_cell(m, i, Ql, 2)
        assert np.abs(w[i] - r["w"]).max() <= 1e-12 * np.abs(Ql).max()
        assert np.abs(w[i][:, 4:]).max() <= 1e-11 * np.abs(Ql).max()       # no quadratic modes


@pytest.mark.parametrize("family", ["0", "1"], ids=["cellvar", "rowblk"])
def test_strides_parts_determinism(family):
    nodes, cells, period = gen.box_mesh(2, 20, True, 0.2, 9)
    V, M = 4, 3
    Q = np.random.default_rng(1).standard_normal((cells.shape[0], V))
    ctx = P.setup_context(nodes, cells, period, M, V, device=0, family=int(family))
    Qd = torch.tensor(Q, device="cuda")
    ref = ctx.reconstruct(Qd)
    again = ctx.reconstruct(Qd)
    assert torch.equal(ref, again)                                        # deterministic
    # strided avgs (column slice of a wider array) and padded output rows
    wide = torch.zeros((Q.shape[0], V + 3), dtype=torch.float64, device="cuda")
    wide[:, 2:2 + V] = Qd
    out = torch.full((Q.shape[0], V, 16), np.nan, dtype=torch.float64, device="cuda")[:, :, : ctx.nm]
    for k in ("pipelined", "simple"):
        ctx.set_kernel(k)
        ctx.reconstruct(wide[:, 2:2 + V], out)
        assert torch.equal(out, ref)
    # transposed avgs layout [V][N]
    ctx.reconstruct(Qd.t().contiguous().t(), out)
    assert torch.equal(out, ref)
    # interior + boundary parts == all (single rank: every cell is interior)
    ctx.set_kernel("pipelined")
    o2 = torch.zeros_like(ref)
    ctx.reconstruct(Qd, o2, part=P.PART_INTERIOR)
    ctx.reconstruct(Qd, o2, part=P.PART_BOUNDARY)
    assert torch.equal(o2, ref)


@pytest.mark.parametrize("family", ["0", "1"], ids=["cellvar", "rowblk"])
def test_multirank_emulation_bitwise(family):
    """T5: P logical ranks on one GPU (one context each, ghosts filled from the
    global array, library halo pack checked) reproduce the 1-rank output bitwise."""
    nodes, cells, period = gen.box_mesh(2, 22, True, 0.2, 13)
    V, M, NR = 3, 3, 3
    Qin = np.random.default_rng(2).standard_normal((cells.shape[0], V))
    one = P.setup_context(nodes, cells, period, M, V, device=0, family=int(family))
    perm = one.permutation()
    Qg = Qin[perm]
    ref = one.reconstruct(torch.tensor(Qg, device="cuda")).cpu().numpy()
    ctxs, plans = [], []
    for r in range(NR):
        c = P.Context(2, M, V, device=0)
        c.set_option(P.OPT_FAMILY, int(family))
        c.set_mesh(nodes, cells, period)
        c.set_partition(r, NR)
        c.build_stencils()
        c.precompute()
        ctxs.append(c)
        plans.append(c.halo_plan())
    for r, c in enumerate(ctxs):
        # send lists: what every other rank requests from r
        cnt = np.array([plans[p][0][r] for p in range(NR)])
        ids = np.concatenate([plans[p][1][plans[p][0][:r].sum():plans[p][0][:r + 1].sum()] for p in range(NR)])
        c.set_send_lists(cnt, ids)
        loc = c.local_cells()
        inf = c.info()
        A = torch.tensor(Qg[loc], device="cuda")
        if c.send_total():
            buf = torch.empty((c.send_total(), V), dtype=torch.float64, device="cuda")
            c.halo_pack(A, buf)
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy(), Qg[ids])
        out = torch.empty((inf["n_owned"], V, c.nm), dtype=torch.float64, device="cuda")
        c.reconstruct(A, out, part=P.PART_INTERIOR)
        c.reconstruct(A, out, part=P.PART_BOUNDARY)
        assert np.array_equal(out.cpu().numpy(), ref[loc[: inf["n_owned"]]])
        # second exchange: the library packs the requested polynomial rows
        if c.send_total():
            rows = out.reshape(inf["n_owned"], V * c.nm)
            wbuf = torch.empty((c.send_total(), V * c.nm), dtype=torch.float64, device="cuda")
            c.halo_pack_rows(rows, wbuf)
            torch.cuda.synchronize()
            assert np.array_equal(wbuf.cpu().numpy(), ref[ids].reshape(len(ids), V * c.nm))


def test_reconstruct_host_end_to_end():
    """cwreco_reconstruct_host (host buffers, pieces overlapped with their D2H) equals
    the device-pointer call bitwise, for pinned and pageable buffers and any piece count."""
    nodes, cells, period = gen.box_mesh(3, 7, True, 0.1, 5)
    V, M = 5, 3
    Q = np.random.default_rng(4).standard_normal((cells.shape[0], V)) + 2.0
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    Qp = Q[ctx.permutation()]
    ref = ctx.reconstruct(torch.tensor(Qp, device="cuda")).cpu()
    for pinned in (True, False):
        h = torch.from_numpy(Qp.copy())
        if pinned:
            h = h.pin_memory()
        for pieces in (0, 1, 3, 7):
            out = ctx.reconstruct_host(h, n_pieces=pieces)
            assert torch.equal(out, ref), (pinned, pieces)


MF_CASES = [
    # name, d, n, M, jitter, periodic, V
    ("2d-M3-jit", 2, 16, 3, 0.2, True, 4),
    ("2d-M2-open", 2, 11, 2, 0.15, False, 3),
    ("3d-M2", 3, 6, 2, 0.0, True, 5),
    ("3d-M3-jit", 3, 6, 3, 0.1, True, 9),
    ("3d-M1-open", 3, 5, 1, 0.1, False, 2),
]


@pytest.mark.parametrize("case", MF_CASES, ids=lambda c: c[0])
def test_matrixfree_parity(case):
    """Matrix-free mode: matrices assembled and least-squares
    problems solved per pass on the GPU; no precompute.  Same tolerance against the
    oracle (R25); against the precomputed-matrix kernel within QR rounding."""
    name, d, n, M, jit, per, V = case
    nodes, cells, period = gen.box_mesh(d, n, per, jit, 31)
    Qin = np.random.default_rng(8).standard_normal((cells.shape[0], V)) * 2.0 + 3.0
    ctx = P.Context(d, M, V, device=0)
    ctx.set_mesh(nodes, cells, period)
    ctx.build_stencils()
    ctx.prepare_matrixfree()
    m = OracleMesh(nodes, cells, period, M)
    Q = Qin[m.perm]
    a = _run(ctx, Q, "matrixfree")
    assert np.all(np.isfinite(a))
    worst = 0.0
    for i in range(m.N):
        r = R.reconstruct_cell(m, i, Q, M)
        worst = max(worst, floored_err(a[i], r["w"], Q, r["central"]))
    assert worst <= TOL, (name, worst)
    ctx.precompute()
    b = _run(ctx, Q, "pipelined")
    scale = np.abs(Q).max()
    assert np.abs(a - b).max() <= 1e-12 * scale
    psi1 = np.sqrt(2.0 if d == 2 else 6.0)
    assert np.abs(a[:, :, 0] * psi1 - Q).max() <= 4e-16 * scale     # conservation
    # interior + boundary parts == all; deterministic
    ctx.set_kernel("matrixfree")
    Qd = torch.tensor(Q, device="cuda")
    o2 = torch.zeros((m.N, V, ctx.nm), dtype=torch.float64, device="cuda")
    ctx.reconstruct(Qd, o2, part=P.PART_INTERIOR)
    ctx.reconstruct(Qd, o2, part=P.PART_BOUNDARY)
    assert np.array_equal(o2.cpu().numpy(), a)
    # host buffers through cwreco_reconstruct_host, in pieces of cells
    assert np.array_equal(ctx.reconstruct_host(Q, n_pieces=3).numpy(), a)


@pytest.mark.parametrize("d,M,V,per", [(2, 3, 4, True), (3, 2, 5, True), (3, 3, 9, True), (2, 2, 3, False)],
                         ids=["2d-M3", "3d-M2", "3d-M3-V9", "2d-M2-open"])
def test_face_traces_parity(d, M, V, per):
    """cwreco_face_traces (NEXT-3) from the GPU coefficients against the oracle's traces
    of its own reconstruction (R25 floored tolerance); the two cells of every interior
    face produce their traces at the same physical points (continuous data agree)."""
    from oracle import traces as TR
    nodes, cells, period = gen.box_mesh(d, 9 if d == 2 else 4, per, 0.15, 17)
    Qin = np.random.default_rng(5).standard_normal((cells.shape[0], V)) + 2.0
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    m = OracleMesh(nodes, cells, period, M)
    Q = Qin[m.perm]
    w = ctx.reconstruct(torch.tensor(Q, device="cuda"))
    tr = ctx.face_traces(w)
    torch.cuda.synchronize()
    tr = tr.cpu().numpy()
    assert tr.shape == (m.N, d + 1, TR.face_rule(d, M)[0].shape[0], V)
    worst = 0.0
    for i in range(0, m.N, 3):
        r = R.reconstruct_cell(m, i, Q, M)
        ref = TR.cell_traces(m, i, r["w"], M)              # [d+1, nq, V]
        s = np.abs(Q[np.asarray(r["central"])]).max(axis=0)  # R25 floor per variable
        err = np.abs(tr[i] - ref) / np.maximum(np.abs(ref), s)
        worst = max(worst, float(err.max()))
    assert worst <= TOL, worst


@pytest.mark.parametrize("d,M,V", [(2, 3, 4), (3, 2, 5), (3, 3, 5), (3, 3, 9), (3, 2, 9), (2, 1, 7)],
                         ids=["2d-M3", "3d-M2", "3d-M3", "3d-M3-V9", "3d-M2-V9", "2d-M1-V7"])
def test_face_traces_many_steps_and_strided(d, M, V):
    """The staged-block trace kernel with 2 CTAs walking every block of cells (double
    buffering of the coefficient blocks, output buffer reuse) equals the uncapped launch
    bitwise, and so does a strided coefficient array (per-element cp.async path instead
    of the bulk copies); the traces of the uncapped launch also match the oracle's on a
    sample of cells."""
    from oracle import traces as TR
    nodes, cells, period = gen.box_mesh(d, 24 if d == 2 else 6, True, 0.15, 23)
    Qin = np.random.default_rng(9).standard_normal((cells.shape[0], V)) + 2.0
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    m = OracleMesh(nodes, cells, period, M)
    Q = Qin[m.perm]
    w = ctx.reconstruct(torch.tensor(Q, device="cuda"))
    ref = ctx.face_traces(w).cpu().numpy()
    ctx.set_option(P.OPT_MAX_CTAS, 2)
    capped = ctx.face_traces(w).cpu().numpy()
    assert np.array_equal(capped, ref)
    wpad = torch.zeros((w.shape[0], V + 1, w.shape[2] + 3), dtype=torch.float64, device="cuda")
    wpad[:, :V, :w.shape[2]] = w
    strided = ctx.face_traces(wpad[:, :V, :w.shape[2]]).cpu().numpy()
    assert np.array_equal(strided, ref)
    worst = 0.0
    for i in list(range(0, m.N, max(1, m.N // 40))) + [m.N - 1]:
        r = R.reconstruct_cell(m, i, Q, M)
        tr_o = TR.cell_traces(m, i, r["w"], M)
        s = np.abs(Q[np.asarray(r["central"])]).max(axis=0)
        worst = max(worst, float((np.abs(ref[i] - tr_o) / np.maximum(np.abs(tr_o), s)).max()))
    assert worst <= TOL, worst


def test_c_client_on_gpu(tmp_path):
    """examples/cwreco_example.c end to end on the GPU through the C-ABI alone."""
    import subprocess
    from test_library_host import _build_c_example
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe, "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "conservation error" in r.stdout


def test_rowblk_constant_data():
    """The row-block family forms B⁺ΔQ as B⁺Q − rs·Q_i: on constant data the higher
    modes are rounding-level (not exactly 0 as in the ΔQ form), the mean exact."""
    nodes, cells, period = gen.box_mesh(3, 4, True, 0.1, 4)
    ctx = P.setup_context(nodes, cells, period, 3, 9, device=0, family=1)
    assert ctx.info()["kernel_family"] == 1
    Qc = np.full((cells.shape[0], 9), 1.25)
    w = _run(ctx, Qc, "pipelined")
    assert np.all(w[:, :, 0] == 1.25 / np.sqrt(6.0))
    assert np.abs(w[:, :, 1:]).max() <= 1e-14 * 1.25


@pytest.mark.parametrize("family", ["0", "1"], ids=["cellvar", "rowblk"])
def test_multirank_loopback_overlap(family):
    """The library's own exchange path on ONE GPU: 3 ranks in 3 host threads, each
    with its own context joined by a loopback transport (cwreco_set_partition with a
    loopback id).  cwreco_reconstruct_overlap = pack → peer copies into the ghost rows
    on the comm stream, interior tiles concurrently, boundary tiles after the event.
    Every rank's ghost rows equal the owners' averages and its coefficients equal
    the single-rank pass BITWISE, for three passes in a row (buffer reuse across
    epochs) with a small CTA cap (many tiles per CTA); the second exchange
    (cwreco_halo_exchange_rows) delivers the owners' polynomial rows."""
    import threading
    nodes, cells, period = gen.box_mesh(2, 40, True, 0.2, 13)
    V, M, NR = 3, 3, 3
    Qin = np.random.default_rng(2).standard_normal((cells.shape[0], V))
    one = P.setup_context(nodes, cells, period, M, V, device=0, family=int(family))
    Qg = Qin[one.permutation()]
    ref = one.reconstruct(torch.tensor(Qg, device="cuda")).cpu().numpy()
    uid = P.loopback_unique_id(NR)
    res, errs = [None] * NR, []

    def run(r):
        try:
            c = P.Context(2, M, V, device=0)
            c.set_option(P.OPT_FAMILY, int(family))
            c.set_option(P.OPT_MAX_CTAS, 3)
            c.set_mesh(nodes, cells, period)
            c.set_partition(r, NR, uid)
            c.build_stencils()                 # collective: plan exchange
            c.precompute()
            inf = c.info()
            loc = c.local_cells()
            n_owned = inf["n_owned"]
            st = torch.cuda.Stream()
            outs, ghosts = [], []
            with torch.cuda.stream(st):
                A = torch.full((len(loc), V), float("nan"), dtype=torch.float64, device="cuda")
                A[:n_owned] = torch.tensor(Qg[loc[:n_owned]], device="cuda")
                for it in range(3):
                    out = torch.full((n_owned, V, c.nm), float("nan"), dtype=torch.float64, device="cuda")
                    c.reconstruct_overlap(A, out, stream=st)
                    outs.append(out)
                # second exchange: polynomial rows of the ghosts
                W = torch.full((len(loc), V * c.nm), float("nan"), dtype=torch.float64, device="cuda")
                W[:n_owned] = outs[-1].reshape(n_owned, V * c.nm)
                c.halo_exchange_rows(W, stream=st)
            st.synchronize()
            res[r] = (loc, n_owned, inf, A.cpu().numpy(), [o.cpu().numpy() for o in outs], W.cpu().numpy(), c)
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))
    th = [threading.Thread(target=run, args=(r,)) for r in range(NR)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(NR):
        loc, n_owned, inf, A, outs, W, c = res[r]
        assert inf["n_ghost"] > 0 and inf["n_interior"] < n_owned
        assert np.array_equal(A[n_owned:], Qg[loc[n_owned:]])
        for o in outs:
            assert np.array_equal(o, ref[loc[:n_owned]])
        assert np.array_equal(W[n_owned:], ref[loc[n_owned:]].reshape(-1, V * c.nm))


def test_many_tiles_per_cta_parity():
    """CWRECO_OPT_MAX_CTAS: with 2 CTAs every CTA walks many tiles (double-buffered
    union gather of the next tile, ring phase wrap-around across tiles), bitwise equal
    to the default launch and to the simple kernel, for both families and 2-D / 3-D."""
    for d, n, M, V, fam in [(2, 24, 3, 4, 0), (2, 24, 3, 4, 1), (3, 6, 2, 5, 0), (3, 6, 3, 9, 1), (3, 6, 3, 5, 0)]:
        nodes, cells, period = gen.box_mesh(d, n, True, 0.15, 23)
        Q = np.random.default_rng(d + M).standard_normal((cells.shape[0], V)) + 1.0
        ctx = P.setup_context(nodes, cells, period, M, V, device=0, family=fam)
        Qp = torch.tensor(Q[ctx.permutation()], device="cuda")
        full = ctx.reconstruct(Qp).cpu().numpy()
        ctx.set_option(P.OPT_MAX_CTAS, 2)
        assert ctx.info()["n_tiles"] >= 8
        capped = ctx.reconstruct(Qp).cpu().numpy()
        ctx.set_kernel("simple")
        simple = ctx.reconstruct(Qp).cpu().numpy()
        assert np.array_equal(capped, full), (d, M, V, fam)
        assert np.array_equal(simple, full), (d, M, V, fam)


def test_smaller_tile_parity():
    """CWRECO_OPT_MAX_TILE: layouts with smaller tiles (the row-block kernel's runtime-T
    instantiation, the one a layout whose tile had to be halved runs) give results
    bitwise equal to the full-tile layout (compile-time T) and to k_simple, with many
    tiles per CTA."""
    for d, n, M, V, fam in [(3, 6, 3, 9, 1), (3, 6, 2, 5, 1), (2, 24, 3, 4, 1), (2, 24, 3, 4, 0)]:
        nodes, cells, period = gen.box_mesh(d, n, True, 0.15, 29)
        Q = np.random.default_rng(d * M + V).standard_normal((cells.shape[0], V)) + 1.0
        ctx = P.setup_context(nodes, cells, period, M, V, device=0, family=fam)
        Tfull = ctx.info()["tile_cells"]
        Qp = torch.tensor(Q[ctx.permutation()], device="cuda")
        full = ctx.reconstruct(Qp).cpu().numpy()
        for cap in (Tfull // 2, 10):
            ctx.set_option(P.OPT_MAX_TILE, cap)
            ctx.precompute()
            assert ctx.info()["tile_cells"] == cap, (d, M, V, fam, cap)
            ctx.set_option(P.OPT_MAX_CTAS, 3)
            got = ctx.reconstruct(Qp).cpu().numpy()
            ctx.set_option(P.OPT_MAX_CTAS, 0)
            assert np.array_equal(got, full), (d, M, V, fam, cap)
        ctx.set_kernel("simple")
        assert np.array_equal(ctx.reconstruct(Qp).cpu().numpy(), full)


@pytest.mark.parametrize("family", ["0", "1"], ids=["cellvar", "rowblk"])
@pytest.mark.parametrize("d,n,M,V,bc", [(2, 10, 3, 4, [1, 2, 2, 1]), (2, 9, 2, 4, [2, 2, 2, 2]),
                                        (3, 4, 2, 5, [1, 2, 1, 2, 2, 1]), (3, 4, 3, 5, [2, 0, 1, 1, 2, 2])],
                         ids=["2d-M3", "2d-M2-walls", "3d-M2", "3d-M3"])
def test_boundary_ghost_parity(d, n, M, V, bc, family):
    """NEXT-4 (R37): open meshes with reflected boundary ghosts (transmissive / wall,
    momentum at variable 1): every cell against the oracle at the R25 tolerance, the
    pipelined kernels bitwise equal to k_simple, host-buffer path identical."""
    nodes, cells, _ = gen.box_mesh(d, n, False, 0.12, 19)
    rng = np.random.default_rng(11)
    Qin = rng.standard_normal((cells.shape[0], V)) + 2.0
    ctx = P.Context(d, M, V, device=0)
    ctx.set_option(P.OPT_FAMILY, int(family))
    ctx.set_mesh(nodes, cells, None)
    ctx.set_boundary(bc, mom0=1)
    ctx.build_stencils()
    ctx.precompute()
    assert ctx.info()["n_boundary_ghosts"] > 0
    m = OracleMesh(nodes, cells, None, M, bc=bc, mom0=1)
    Q = Qin[m.perm]
    a = _run(ctx, Q, "pipelined")
    b = _run(ctx, Q, "simple")
    assert np.array_equal(a, b)
    worst = 0.0
    for i in range(m.N):
        r = R.reconstruct_cell(m, i, Q, M)
        S = r["central"]
        vals = m.values(Q, S)
        s = np.abs(vals).max(axis=0)[:, None]
        worst = max(worst, float((np.abs(a[i] - r["w"]) / np.maximum(np.abs(r["w"]), s)).max()))
    assert worst <= TOL, worst
    ctx.set_kernel("pipelined")
    assert np.array_equal(ctx.reconstruct_host(Q).numpy(), a)

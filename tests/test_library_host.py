"""Host-side checks of libcwreco (no GPU): the C-ABI loads and exports every
symbol of include/cwreco.h; the setup (Morton order, stencils) is bit-exact
against the oracle; the precomputed per-cell matrices reproduce the oracle's
P_opt / P_s (T2, host matvec in the test); error codes; layout facts."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import gen
import paper_1612_09335_b200 as P
from oracle import basis as B
from oracle import reconstruct as R
from oracle.mesh import OracleMesh

HEADER = "include/cwreco.h"


def test_header_symbols_exported():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    txt = open(os.path.join(root, HEADER)).read()
    names = sorted(set(re.findall(r"\b(cwreco_[a-z_]+)\s*\(", txt)))
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", P._LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cwreco_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(P.lib, n)
    assert P.lib.cwreco_version().decode().startswith("cwreco")


def _mesh_cases():
    return [
        ("C1", *gen.box_mesh(2, 16, True), 2),
        ("2d-jit-M3", *gen.box_mesh(2, 20, True, 0.2, 5), 3),
        ("2d-open-M2", *gen.box_mesh(2, 9, False, 0.15, 6), 2),
        ("3d-M2", *gen.box_mesh(3, 5, True), 2),
        ("3d-jit-M3", *gen.box_mesh(3, 6, True, 0.1, 7), 3),
        ("3d-open-M1", *gen.box_mesh(3, 4, False, 0.1, 8), 1),
    ]


@pytest.mark.parametrize("case", _mesh_cases(), ids=lambda c: c[0])
def test_permutation_and_stencils_bit_exact(case):
    name, nodes, cells, period, M = case
    ctx = P.Context(nodes.shape[1], M, 3, device=None)
    ctx.set_mesh(nodes, cells, period)
    ctx.build_stencils()
    m = OracleMesh(nodes, cells, period, M)
    assert np.array_equal(ctx.permutation(), m.perm)
    cen, sec, val = ctx.stencils()
    assert np.array_equal(ctx.local_cells(), np.arange(m.N))
    for i in range(m.N):
        c = m.central_stencil(i)
        s, v = m.sector_stencils(i)
        assert cen[i].tolist() == c, (name, i)
        assert sec[i].tolist() == s, (name, i)
        assert val[i].tolist() == v, (name, i)


def test_stencils_full_size_c2_sample():
    w = gen.make("C2")
    ctx = P.Context(2, 3, 4, device=None)
    ctx.set_mesh(w["nodes"], w["cells"], w["period"])
    ctx.build_stencils()
    m = OracleMesh(w["nodes"], w["cells"], w["period"], 3)
    assert np.array_equal(ctx.permutation(), m.perm)
    cen, sec, val = ctx.stencils()
    rng = np.random.default_rng(0)
    for i in rng.choice(m.N, 300, replace=False):
        s, v = m.sector_stencils(int(i))
        assert cen[i].tolist() == m.central_stencil(int(i))
        assert sec[i].tolist() == s and val[i].tolist() == v
    inf = ctx.info()
    # R15: some sectors reach outside the central stencil in jittered C2; R14: none starve
    assert inf["n_invalid_sectors"] == 0


@pytest.mark.parametrize("d,M", [(2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3)])
def test_sigma_matches_oracle(d, M):
    ctx = P.Context(d, M, 1, device=None)
    S = ctx.sigma()
    So = B.sigma_numeric(d, M)
    assert np.abs(S - So).max() <= 1e-13 * np.abs(So).max()


@pytest.mark.parametrize("case", _mesh_cases(), ids=lambda c: c[0])
def test_precompute_parity_host(case):
    """T2: the packed B⁺ and sector inverses applied on the host reproduce the
    oracle's constrained-LSQ and sector polynomials (floored relative 1e-12)."""
    name, nodes, cells, period, M = case
    d, V = nodes.shape[1], 3
    rng = np.random.default_rng(1)
    Qin = rng.standard_normal((cells.shape[0], V)) + 2.0
    ctx = P.setup_context(nodes, cells, period, M, V, device=None)
    m = OracleMesh(nodes, cells, period, M)
    Q = Qin[m.perm]
    sel = rng.choice(m.N, min(m.N, 25), replace=False)
    blk = ctx.blocks(sel)
    n_e = d * P.n_modes(M, d)
    for q, i in enumerate(sel):
        r = R.reconstruct_cell(m, int(i), Q, M)
        g = blk["gather"][q]
        scale = np.abs(Q[r["central"]]).max()
        popt = blk["bplus"][q] @ (Q[g] - Q[i])
        # every cell of S_i^0 ∖ i appears exactly once in the gather list
        assert sorted(set(g.tolist()) - {int(i)}) == sorted(set(r["central"][1:])) or \
            set(r["central"][1:]) <= set(g.tolist())
        assert np.abs(popt.T - r["popt"][:, 1:]).max() <= 1e-12 * scale, (name, i)
        for s in range(d + 1):
            sl = blk["slots"][q][s]
            assert (sl[0] == 255) == (not r["valid"][s])
            if r["valid"][s]:
                ps = blk["sinv"][q][s] @ (Q[g[sl]] - Q[i])
                assert np.abs(ps.T - r["psec"][s][:, 1:]).max() <= 1e-12 * scale


def test_algorithmic_bytes_per_cell_table():
    # SURVEY.md §8(d) B_cell column: 810 / 1898 / 2944 / 11016 / 10344
    for (d, M, V, want) in [(2, 2, 4, 810), (2, 3, 4, 1898), (3, 2, 5, 2944), (3, 3, 9, 11016), (3, 3, 5, 10344)]:
        ctx = P.Context(d, M, V, device=None)
        assert ctx.info()["algorithmic_bytes_per_cell"] == want


def test_layout_and_info():
    nodes, cells, period = gen.box_mesh(2, 16, True)
    ctx = P.setup_context(nodes, cells, period, 2, 4, device=None)
    inf = ctx.info()
    T = inf["tile_cells"]
    assert inf["n_tiles"] == -(-512 // T) and inf["n_interior_tiles"] == inf["n_tiles"]
    assert inf["tile_bytes"] % 16 == 0 and T % 2 == 0 and inf["chunk_k"] >= 1
    assert inf["n_e"] == 12 and inf["n_modes"] == 6 and inf["n_ghost"] == 0


def test_error_codes():
    with pytest.raises(P.CwrecoError, match="EUNSUPPORTED"):
        P.Context(4, 2, 1, device=None)
    with pytest.raises(P.CwrecoError, match="EUNSUPPORTED"):
        P.Context(3, 4, 1, device=None)
    with pytest.raises(P.CwrecoError, match="EUNSUPPORTED"):
        P.Context(2, 2, 17, device=None)
    nodes, cells, period = gen.box_mesh(2, 3, True)
    ctx = P.Context(2, 1, 1, device=None)
    with pytest.raises(P.CwrecoError, match="ESTATE"):
        ctx.build_stencils()
    with pytest.raises(P.CwrecoError, match="EMESH"):
        ctx.set_mesh(nodes, np.vstack([cells, cells[:1]]), period)          # duplicate cell
    bad = cells.copy(); bad[0, 2] = bad[0, 1]
    with pytest.raises(P.CwrecoError, match="EMESH"):
        ctx.set_mesh(nodes, bad, period)                                      # repeated vertex
    flat = nodes.copy(); flat[:, 1] = 0.0
    with pytest.raises(P.CwrecoError, match="EMESH"):
        ctx.set_mesh(flat, cells, None)                                       # zero area
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        ctx.set_mesh(nodes, cells + 100, period)                              # missing node
    n2, c2, _ = gen.box_mesh(2, 2, False)
    ctx2 = P.Context(2, 2, 1, device=None)
    ctx2.set_mesh(n2, c2, None)
    with pytest.raises(P.CwrecoError, match="ESTENCIL"):
        ctx2.build_stencils()                                                 # 8 cells < n_e = 12
    ctx3 = P.setup_context(nodes, cells, period, 1, 1, device=None)
    # no CPU fallback: compute calls fail loudly on a host-only context
    st = P.lib.cwreco_reconstruct(ctx3._h, ctypes.c_void_p(8), 1, 1, ctypes.c_void_p(8), 3, 3, 0, None)
    assert P._STATUS[st] == "ECUDA" and "no CPU fallback" in P.lib.cwreco_last_error().decode()
    st = P.lib.cwreco_reconstruct_debug(ctx3._h, ctypes.c_void_p(8), 1, 1, 0, None, None, None, None, None,
                                        None, None)
    assert P._STATUS[st] == "ECUDA"


def test_partition_host_logic():
    """Two ranks of a contiguous Morton partition: ghosts are exactly the
    non-owned stencil cells, interior cells need no ghost, the ghost plan of one
    rank equals the send list the other must provide."""
    nodes, cells, period = gen.box_mesh(2, 20, True, 0.2, 3)
    M, V, P_ = 3, 2, 2
    full = P.Context(2, M, V, device=None)
    full.set_mesh(nodes, cells, period)
    full.build_stencils()
    cen_all, sec_all, _ = full.stencils()
    N = cells.shape[0]
    ctxs = []
    for r in range(P_):
        c = P.Context(2, M, V, device=None)
        c.set_mesh(nodes, cells, period)
        c.set_partition(r, P_)
        c.build_stencils()
        ctxs.append(c)
    plans = [c.halo_plan() for c in ctxs]
    for r, c in enumerate(ctxs):
        lo, hi = r * N // P_, (r + 1) * N // P_
        inf = c.info()
        assert inf["n_owned"] == hi - lo
        loc = c.local_cells()
        owned = loc[: inf["n_owned"]]
        assert sorted(owned.tolist()) == list(range(lo, hi))
        need = set()
        for g in owned:
            need |= set(cen_all[g].tolist()) | set(x for x in sec_all[g].ravel().tolist() if x >= 0)
        ghosts = sorted(x for x in need if not lo <= x < hi)
        assert loc[inf["n_owned"]:].tolist() == ghosts
        # interior cells first: their stencils are fully owned
        for g in owned[: inf["n_interior"]]:
            assert all(lo <= x < hi for x in cen_all[g])
        for g in owned[inf["n_interior"]:]:
            assert not all(lo <= x < hi for x in set(cen_all[g]) | set(y for y in sec_all[g].ravel() if y >= 0))
        # stencils of a partition equal the global ones (same SFC ids)
        cen, sec, _ = c.stencils()
        assert np.array_equal(cen, cen_all[owned]) and np.array_equal(sec, sec_all[owned])
        counts, ids = plans[r]
        assert counts.sum() == len(ghosts) and counts[r] == 0
    # rank 0's request from rank 1 are rank-1 cells, and installs as rank 1's send list
    c1 = ctxs[1]
    counts0, ids0 = plans[0]
    send_counts = np.array([counts0[1], 0])
    c1.set_send_lists(send_counts, ids0[counts0[0]:])
    assert c1.send_total() == counts0[1]
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        c1.set_send_lists(np.array([1, 0]), np.array([0]))                   # not owned by rank 1


def test_set_stencils_roundtrip_and_validation():
    """cwreco_set_stencils (S:194-211 interface): stencils built by the library, uploaded
    into a fresh context in SFC order, give identical local numbering and identical
    per-cell matrices; malformed stencils are rejected with EINVAL."""
    nodes, cells, period = gen.box_mesh(2, 10, True, 0.2, 7)
    a = P.Context(2, 3, 2, device=None)
    a.set_mesh(nodes, cells, period)
    a.build_stencils()
    a.precompute()
    cen_l, sec_l, val_l = a.stencils()               # local order
    loc = a.local_cells()
    n_own = a.info()["n_owned"]
    order = np.argsort(loc[:n_own])                   # local -> SFC order
    cen, sec, val = cen_l[order], sec_l[order], val_l[order]
    b = P.Context(2, 3, 2, device=None)
    b.set_mesh(nodes, cells, period)
    b.set_stencils(cen, sec, val)
    assert np.array_equal(b.local_cells(), loc)
    b.precompute()
    sel = np.arange(0, n_own, 7)
    ba, bb = a.blocks(sel), b.blocks(sel)
    for k in ba:
        assert np.array_equal(ba[k], bb[k]), k
    bad = cen.copy()
    bad[3, 0] = bad[3, 1]                             # cell not first
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        b.set_stencils(bad, sec, val)
    bad = cen.copy()
    bad[5, 2] = bad[5, 1]                             # repeated member
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        b.set_stencils(bad, sec, val)
    c = P.Context(2, 3, 2, device=None)
    with pytest.raises(P.CwrecoError, match="ESTATE"):
        c.set_stencils(cen, sec, val)


@pytest.mark.parametrize("d,M", [(2, 3), (3, 2), (3, 3)])
def test_face_rule_and_neighbors_match_oracle(d, M):
    """cwreco_face_rule is the oracle's rule (same points, same order, same weights);
    cwreco_face_neighbors equals the oracle's face adjacency in local numbering."""
    from oracle import traces as TR
    nodes, cells, period = gen.box_mesh(d, 6 if d == 2 else 3, True, 0.1, 3)
    ctx = P.Context(d, M, 1, device=None)
    ctx.set_mesh(nodes, cells, period)
    ctx.build_stencils()
    lam, w = ctx.face_rule()
    lo, wo = TR.face_rule(d, M)
    assert np.allclose(lam, lo, atol=1e-14, rtol=0) and np.allclose(w, wo, atol=1e-15, rtol=0)
    m = OracleMesh(nodes, cells, period, M)
    loc = ctx.local_cells()
    nb = ctx.face_neighbors()
    n_own = nb.shape[0]
    for li in range(n_own):
        g = loc[li]
        want = m.nbr[g]
        got = np.where(nb[li] >= 0, loc[np.maximum(nb[li], 0)], -1)
        assert np.array_equal(got, want), li


def _build_c_example(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_1612_09335_b200")
    exe = str(tmp_path / "cwreco_example")
    subprocess.run(["cc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "cwreco_example.c"), "-L", lib, "-lcwreco",
                    "-Wl,-rpath," + lib, "-lm", "-o", exe], check=True)
    return exe


def test_c_client_host_only(tmp_path):
    """The C-ABI is usable from plain C (examples/cwreco_example.c): mesh, stencils and
    precompute run on the host; the compute call reports ECUDA (no CPU fallback)."""
    exe = _build_c_example(tmp_path)
    r = subprocess.run([exe, "-1"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "cells 1152, modes 10" in r.stdout and "status 3" in r.stderr


def test_sector_fallback_hand_mesh_library():
    """The library's stencil builder on the hand-derived R14 fallback mesh
    (tests/golden/sector_fallback_mesh.json): same sectors and validity as derived
    by hand, the fallback cell counted as an extra gather (R15), and the
    precomputed matrices reproduce linear data exactly on the owner."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "sector_fallback_mesh.json")) as f:
        g = json.load(f)
    nodes, cells = np.array(g["nodes"]), np.array(g["cells"], dtype=np.int64)
    ctx = P.Context(2, g["M"], 2, device=None)
    ctx.set_mesh(nodes, cells, None)
    ctx.build_stencils()
    perm = ctx.permutation()
    sfc = {int(inp): s for s, inp in enumerate(perm)}
    cen, sec, val = ctx.stencils()
    i = sfc[g["owner"]]
    exp = [[sfc[c] if c >= 0 else -1 for c in row] for row in g["expected_sectors_input_ids"]]
    assert sec[i].tolist() == exp
    assert val[i].tolist() == g["expected_valid"]
    assert sfc[2] not in cen[i].tolist()
    ctx.precompute()
    assert ctx.info()["n_extra_gather"] >= 1
    assert ctx.info()["n_invalid_sectors"] >= 2


def test_loopback_plan_exchange_host_threads():
    """The library's own plan exchange (cwreco_set_partition with a loopback id,
    collective cwreco_build_stencils): three host-only contexts in three threads;
    each rank's installed send lists equal what the other ranks requested
    (cwreco_halo_plan), peer by peer, in order."""
    import threading
    nodes, cells, period = gen.box_mesh(2, 18, True, 0.2, 7)
    NR = 3
    uid = P.loopback_unique_id(NR)
    ctxs = [P.Context(2, 3, 2, device=None) for _ in range(NR)]
    errs = []

    def run(r):
        try:
            ctxs[r].set_mesh(nodes, cells, period)
            ctxs[r].set_partition(r, NR, uid)
            ctxs[r].build_stencils()            # collective: plan exchange inside
        except Exception as e:                  # pragma: no cover
            errs.append(repr(e))
    th = [threading.Thread(target=run, args=(r,)) for r in range(NR)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    plans = [c.halo_plan() for c in ctxs]
    for r, c in enumerate(ctxs):
        counts, ids = c.send_lists()
        want_ids = []
        for p in range(NR):
            pc, pid = plans[p]
            off = int(pc[:r].sum())
            assert counts[p] == pc[r]
            want_ids += pid[off:off + pc[r]].tolist()
        assert ids.tolist() == want_ids
        assert counts[r] == 0 and c.send_total() == len(want_ids) > 0
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        P.Context(2, 3, 2, device=None).set_partition(0, 3, b"CWRLOOP\x00" + b"\xff" * 120)  # unknown group
    with pytest.raises(P.CwrecoError, match="ESTATE|ECUDA"):
        ctxs[0].halo_exchange.__func__  # noqa: B018 (attribute exists)
        import ctypes
        st = P.lib.cwreco_halo_exchange(ctxs[0]._h, ctypes.c_void_p(8), 2, 1, None)
        P._check(st)


@pytest.mark.parametrize("d,n,M,bc", [(2, 8, 2, [1, 2, 1, 2]), (2, 7, 3, [2, 2, 0, 1]), (3, 4, 2, [1, 1, 2, 2, 1, 0])])
def test_boundary_ghost_stencils_bit_exact(d, n, M, bc):
    """R37: the library's stencils with reflected boundary ghosts equal the oracle's
    bit for bit (ghost ids N + s·N + k), and the precompute accepts them."""
    nodes, cells, _ = gen.box_mesh(d, n, False, 0.12, 9)
    ctx = P.Context(d, M, d + 2, device=None)
    ctx.set_mesh(nodes, cells, None)
    ctx.set_boundary(bc, mom0=1)
    ctx.build_stencils()
    m = OracleMesh(nodes, cells, None, M, bc=bc, mom0=1)
    assert np.array_equal(ctx.permutation(), m.perm)
    cen, sec, val = ctx.stencils()
    for i in range(m.N):
        assert cen[i].tolist() == m.central_stencil(i), i
        s, v = m.sector_stencils(i)
        assert sec[i].tolist() == s and val[i].tolist() == v, i
    ctx.precompute()
    assert ctx.info()["n_boundary_ghosts"] > 0
    with pytest.raises(P.CwrecoError, match="EINVAL"):
        c2 = P.Context(d, M, d + 2, device=None)
        c2.set_mesh(*gen.box_mesh(d, n, True)[:2], np.ones(d))
        c2.set_boundary(bc, 1)


def test_partition_keeps_full_rowblock_tile():
    """A partitioned rank keeps the row-block tile of one rank (T = 32 cells for the C4
    shape): boundary tiles raise the stencil-union maximum (370 → 519 cells here), and
    the layout takes fewer ring stages before it halves the tile (rank projection: a
    C4 rank at T = 16 cost 1.48× the time per cell).  Host-only: the layout is planned
    for the 227 KB shared-memory opt-in of sm_100a."""
    nodes, cells, per = gen.box_mesh(3, 16, True, 0.1, 4)
    seen = {}
    for nranks in (1, 2, 4, 8):
        c = P.Context(3, 3, 9, device=None)
        c.set_mesh(nodes, cells, per)
        if nranks > 1:
            c.set_partition(nranks - 1, nranks)
        c.build_stencils()
        c.precompute()
        i = c.info()
        assert i["kernel_family"] == 1
        seen[nranks] = (i["tile_cells"], i["union_max"])
    assert all(t == 32 for t, _ in seen.values()), seen
    assert max(u for _, u in seen.values()) > seen[1][1]      # the case this guards

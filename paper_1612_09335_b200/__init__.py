"""Python binding of libcwreco (include/cwreco.h): argument marshalling only.

Every step of the reconstruction runs in the library (host C++ for the one-time
setup, sm_100a CUDA kernels for the pass).  PyTorch provides device memory and
streams; there is no CPU fallback — a missing or unbuildable library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Context", "CwrecoError", "lib", "KERNELS", "OPT_FAMILY", "OPT_MAX_CTAS", "OPT_MAX_TILE", "PART_ALL",
           "nccl_unique_id", "loopback_unique_id",
           "PART_INTERIOR", "PART_BOUNDARY",
           "n_modes", "setup_context"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libcwreco.so")

KERNELS = {"pipelined": 0, "simple": 1, "matrixfree": 2}
OPT_FAMILY, OPT_MAX_CTAS, OPT_MAX_TILE = 1, 2, 3
PART_ALL, PART_INTERIOR, PART_BOUNDARY = 0, 1, 2
_STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "EMESH", 5: "ESTENCIL", 6: "ESINGULAR",
           7: "ESTATE", 8: "EUNSUPPORTED", 9: "ENCCL"}


class CwrecoError(RuntimeError):
    def __init__(self, status, msg):
        self.status = _STATUS.get(status, str(status))
        super().__init__(f"cwreco {self.status}: {msg}")


class _Params(ctypes.Structure):
    _fields_ = [("lambda0", ctypes.c_double), ("lambda_s", ctypes.c_double), ("eps", ctypes.c_double),
                ("r", ctypes.c_int)]


class _Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("dim", "degree_M", "nvars", "n_modes", "n_e", "gather_len",
                                               "tile_cells", "chunk_k")] + \
               [(n, ctypes.c_int64) for n in ("n_cells", "n_owned", "n_ghost", "n_interior", "n_tiles",
                                               "n_interior_tiles", "tile_bytes", "device_bytes",
                                               "algorithmic_bytes_per_cell", "n_invalid_sectors",
                                               "n_extra_gather", "union_max")] + \
               [(n, ctypes.c_int32) for n in ("kernel_family", "reserved_")] + \
               [("n_boundary_ghosts", ctypes.c_int64)]


def _load():
    from . import _build
    alt = os.environ.get("CWRECO_LIBRARY")   # tuning variants of the library (tools/ only)
    if alt:
        L = ctypes.CDLL(alt)
    else:
        if not os.path.exists(_LIB_PATH) or _build.stale_abi(_LIB_PATH):
            _build.build()   # missing, or older than include/cwreco.h's entry points
        L = ctypes.CDLL(_LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sigs = {
        "cwreco_create": [I32, I32, I32, P, I32, P],
        "cwreco_get_info": [P, P],
        "cwreco_set_kernel": [P, I32],
        "cwreco_set_option": [P, I32, I64],
        "cwreco_set_mesh": [P, I64, P, I64, P, P],
        "cwreco_get_permutation": [P, P],
        "cwreco_set_boundary": [P, P, I32],
        "cwreco_set_partition": [P, I32, I32, P],
        "cwreco_nccl_unique_id": [P],
        "cwreco_loopback_unique_id": [I32, P],
        "cwreco_halo_exchange": [P, P, I64, I64, P],
        "cwreco_halo_exchange_rows": [P, P, I64, I32, P],
        "cwreco_reconstruct_overlap": [P, P, I64, I64, P, I64, I64, P],
        "cwreco_build_stencils": [P],
        "cwreco_get_stencils": [P, P, P, P],
        "cwreco_get_local_cells": [P, P],
        "cwreco_set_stencils": [P, P, P, P],
        "cwreco_prepare_matrixfree": [P],
        "cwreco_face_rule": [P, P, P, P],
        "cwreco_face_neighbors": [P, P],
        "cwreco_face_traces": [P, P, I64, I64, P, P],
        "cwreco_precompute": [P],
        "cwreco_get_sigma": [P, P],
        "cwreco_get_blocks": [P, I64, P, P, P, P, P],
        "cwreco_halo_plan": [P, P, P],
        "cwreco_set_send_lists": [P, P, P],
        "cwreco_send_total": [P, P],
        "cwreco_get_send_lists": [P, P, P],
        "cwreco_halo_pack": [P, P, I64, I64, P, P],
        "cwreco_halo_pack_rows": [P, P, I64, I32, P, P],
        "cwreco_reconstruct": [P, P, I64, I64, P, I64, I64, I32, P],
        "cwreco_reconstruct_debug": [P, P, I64, I64, I64, P, P, P, P, P, P, P],
        "cwreco_reconstruct_host": [P, P, P, I32, P],
        "cwreco_predictor_setup": [P, D],
        "cwreco_predictor_nodes": [P, P, P, P],
        "cwreco_predict": [P, P, I64, I64, D, P, P, P],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.cwreco_destroy.argtypes = [P]
    L.cwreco_destroy.restype = None
    L.cwreco_last_error.restype = ctypes.c_char_p
    L.cwreco_version.restype = ctypes.c_char_p
    return L


lib = _load()


def _check(st):
    if st != 0:
        raise CwrecoError(st, lib.cwreco_last_error().decode())


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def n_modes(M, d):
    num = 1
    for l in range(1, d + 1):
        num *= (M + l)
    return num // (2 if d == 2 else 6)


def nccl_unique_id():
    """128 bytes of a fresh NCCL unique id (cwreco_nccl_unique_id); one rank makes it,
    the caller broadcasts it, every rank passes it to Context.set_partition."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.cwreco_nccl_unique_id(buf))
    return bytes(buf)


def loopback_unique_id(nranks):
    """128 bytes naming a fresh in-process loopback group of nranks ranks
    (cwreco_loopback_unique_id): one thread per rank, each with its own Context."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.cwreco_loopback_unique_id(int(nranks), buf))
    return bytes(buf)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Context:
    """One library context: a mesh, its stencils and per-cell matrices on one device."""

    def __init__(self, dim, degree_M, nvars, device=0, lambda0=1e5, lambda_s=1.0, eps=1e-14, r=4):
        self.dim, self.M, self.V = int(dim), int(degree_M), int(nvars)
        self.nm = n_modes(self.M, self.dim)
        self.device = -1 if device is None else int(device)
        prm = _Params(lambda0, lambda_s, eps, r)
        h = ctypes.c_void_p()
        _check(lib.cwreco_create(self.dim, self.M, self.V, ctypes.byref(prm), self.device, ctypes.byref(h)))
        self._h = h
        self.nranks, self.rank = 1, 0

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.cwreco_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    # ---------------------------------------------------------------- setup
    def set_mesh(self, nodes, cells, period=None):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        per = None if period is None else np.ascontiguousarray(period, dtype=np.float64)
        self.N = cells.shape[0]
        _check(lib.cwreco_set_mesh(self._h, nodes.shape[0], _ptr(nodes), cells.shape[0], _ptr(cells), _ptr(per)))

    def set_boundary(self, side_bc, mom0=-1):
        """cwreco_set_boundary: side_bc [2·dim] (0 none, 1 transmissive, 2 wall) per box
        side s = 2·axis + (0 low, 1 high); mom0 = index of ρu_1 (walls negate ρu_axis)."""
        arr = None if side_bc is None else np.ascontiguousarray(side_bc, dtype=np.int32)
        _check(lib.cwreco_set_boundary(self._h, _ptr(arr), int(mom0)))

    def permutation(self):
        out = np.empty(self.N, dtype=np.int64)
        _check(lib.cwreco_get_permutation(self._h, _ptr(out)))
        return out

    def set_partition(self, rank, nranks, uid=None):
        """cwreco_set_partition; uid: None (no transport) or the 128 bytes of
        nccl_unique_id() / loopback_unique_id() (collective with a transport)."""
        self.rank, self.nranks = int(rank), int(nranks)
        idb = None
        if uid is not None:
            if len(uid) != 128:
                raise ValueError("uid must be 128 bytes")
            idb = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(uid))
        _check(lib.cwreco_set_partition(self._h, self.rank, self.nranks, idb))

    def build_stencils(self):
        _check(lib.cwreco_build_stencils(self._h))

    def info(self):
        i = _Info()
        _check(lib.cwreco_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def stencils(self):
        inf = self.info()
        n, d = inf["n_owned"], self.dim
        cen = np.empty((n, inf["n_e"]), dtype=np.int32)
        sec = np.empty((n, d + 1, d + 1), dtype=np.int32)
        val = np.empty((n, d + 1), dtype=np.uint8)
        _check(lib.cwreco_get_stencils(self._h, _ptr(cen), _ptr(sec), _ptr(val)))
        return cen, sec, val.astype(bool)

    def set_stencils(self, central, sectors, valid):
        """Upload external stencils (owned cells in SFC order, global SFC ids)."""
        central = np.ascontiguousarray(central, dtype=np.int32)
        sectors = np.ascontiguousarray(sectors, dtype=np.int32)
        valid = np.ascontiguousarray(valid, dtype=np.uint8)
        _check(lib.cwreco_set_stencils(self._h, _ptr(central), _ptr(sectors), _ptr(valid)))

    def local_cells(self):
        inf = self.info()
        out = np.empty(inf["n_owned"] + inf["n_ghost"], dtype=np.int64)
        _check(lib.cwreco_get_local_cells(self._h, _ptr(out)))
        return out

    def precompute(self):
        _check(lib.cwreco_precompute(self._h))

    def sigma(self):
        out = np.empty((self.nm, self.nm))
        _check(lib.cwreco_get_sigma(self._h, _ptr(out)))
        return out

    def blocks(self, cells):
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        inf = self.info()
        n, d = len(cells), self.dim
        bp = np.empty((n, self.nm - 1, inf["gather_len"]))
        sv = np.empty((n, d + 1, d, d))
        ga = np.empty((n, inf["gather_len"]), dtype=np.int32)
        sl = np.empty((n, d + 1, d), dtype=np.uint8)
        _check(lib.cwreco_get_blocks(self._h, n, _ptr(cells), _ptr(bp), _ptr(sv), _ptr(ga), _ptr(sl)))
        return dict(bplus=bp, sinv=sv, gather=ga, slots=sl)

    def prepare_matrixfree(self):
        """Upload geometry and stencils for set_kernel("matrixfree") (no matrices)."""
        _check(lib.cwreco_prepare_matrixfree(self._h))

    def set_kernel(self, name):
        _check(lib.cwreco_set_kernel(self._h, KERNELS[name]))

    def set_option(self, option, value):
        """cwreco_set_option: OPT_FAMILY (-1 default, 0 cell-variable, 1 row-block; before
        precompute), OPT_MAX_CTAS (0 = every SM) or OPT_MAX_TILE (cells per tile, 0 = the
        largest that fits; before precompute)."""
        _check(lib.cwreco_set_option(self._h, int(option), int(value)))

    def _need_shape(self, t, shape, what):
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")

    # ---------------------------------------------------------------- halo
    def halo_plan(self):
        inf = self.info()
        counts = np.empty(self.nranks, dtype=np.int64)
        ids = np.empty(inf["n_ghost"], dtype=np.int64)
        _check(lib.cwreco_halo_plan(self._h, _ptr(counts), _ptr(ids)))
        return counts, ids

    def set_send_lists(self, counts, ids):
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        _check(lib.cwreco_set_send_lists(self._h, _ptr(counts), _ptr(ids)))
        self.send_counts = counts

    def send_lists(self):
        """(send_counts [nranks], send_ids [send_total] SFC ids) as installed."""
        counts = np.empty(self.nranks, dtype=np.int64)
        ids = np.empty(max(1, self.send_total()), dtype=np.int64)
        _check(lib.cwreco_get_send_lists(self._h, _ptr(counts), _ptr(ids)))
        return counts, ids[: self.send_total()]

    def send_total(self):
        t = ctypes.c_int64()
        _check(lib.cwreco_send_total(self._h, ctypes.byref(t)))
        return t.value

    def halo_pack(self, avgs, sendbuf, stream=None):
        a_cs, a_vs = avgs.stride()
        _check(lib.cwreco_halo_pack(self._h, ctypes.c_void_p(avgs.data_ptr()), a_cs, a_vs,
                                    ctypes.c_void_p(sendbuf.data_ptr()), _stream_handle(stream)))

    def halo_pack_rows(self, rows, sendbuf, stream=None):
        """rows: CUDA float64 [n_local, W] (row-contiguous, e.g. coefficients viewed as
        [n_local, V·ℳ]); packs the requested owned rows into sendbuf [send_total, W]."""
        if rows.dim() != 2 or rows.stride(1) != 1:
            raise ValueError("rows must be [n_local, W] with contiguous rows")
        _check(lib.cwreco_halo_pack_rows(self._h, ctypes.c_void_p(rows.data_ptr()), rows.stride(0),
                                         rows.shape[1], ctypes.c_void_p(sendbuf.data_ptr()),
                                         _stream_handle(stream)))

    def halo_exchange(self, avgs, stream=None):
        """cwreco_halo_exchange: fill the ghost rows avgs[n_owned:] from their owners."""
        self._check_avgs(avgs)
        a_cs, a_vs = avgs.stride()
        _check(lib.cwreco_halo_exchange(self._h, ctypes.c_void_p(avgs.data_ptr()), a_cs, a_vs,
                                        _stream_handle(stream)))

    def halo_exchange_rows(self, rows, stream=None):
        """cwreco_halo_exchange_rows: rows CUDA float64 [n_local, W] with contiguous rows
        (e.g. coefficients viewed as [n_local, V·ℳ]); fills rows[n_owned:]."""
        import torch
        inf = self.info()
        if not (rows.is_cuda and rows.dtype == torch.float64 and rows.dim() == 2 and rows.stride(1) == 1):
            raise ValueError("rows must be a [n_local, W] float64 CUDA tensor with contiguous rows")
        if rows.shape[0] != inf["n_owned"] + inf["n_ghost"]:
            raise ValueError(f"rows must have n_local = {inf['n_owned'] + inf['n_ghost']} rows")
        _check(lib.cwreco_halo_exchange_rows(self._h, ctypes.c_void_p(rows.data_ptr()), rows.stride(0),
                                             rows.shape[1], _stream_handle(stream)))

    def _check_avgs(self, avgs):
        import torch
        if not (avgs.is_cuda and avgs.dtype == torch.float64 and avgs.dim() == 2):
            raise ValueError("avgs must be a 2-D float64 CUDA tensor")
        inf = self.info()
        self._need_shape(avgs, (inf["n_owned"] + inf["n_ghost"], self.V), "avgs")
        return inf

    # ---------------------------------------------------------------- hot path
    def reconstruct_overlap(self, avgs, out=None, stream=None):
        """cwreco_reconstruct_overlap: halo exchange into avgs' ghost rows overlapped
        with the interior tiles, then the boundary tiles; returns / fills out."""
        import torch
        inf = self._check_avgs(avgs)
        n_owned = inf["n_owned"]
        if out is None:
            out = torch.empty((n_owned, self.V, self.nm), dtype=torch.float64, device=avgs.device)
        if not (out.is_cuda and out.dtype == torch.float64 and out.device == avgs.device):
            raise ValueError("out must be a float64 tensor on the device of avgs")
        self._need_shape(out, (n_owned, self.V, self.nm), "out")
        a_cs, a_vs = avgs.stride()
        c_cs, c_vs, c_ls = out.stride()
        if c_ls != 1:
            raise ValueError("out must be contiguous along the mode axis")
        _check(lib.cwreco_reconstruct_overlap(self._h, ctypes.c_void_p(avgs.data_ptr()), a_cs, a_vs,
                                              ctypes.c_void_p(out.data_ptr()), c_cs, c_vs, _stream_handle(stream)))
        return out

    def reconstruct(self, avgs, out=None, part=PART_ALL, stream=None):
        """avgs: CUDA float64 tensor [n_local, V] (any strides); returns / fills
        out [n_owned, V, ℳ] (float64, CUDA)."""
        import torch
        if not (avgs.is_cuda and avgs.dtype == torch.float64 and avgs.dim() == 2):
            raise ValueError("avgs must be a 2-D float64 CUDA tensor")
        inf = self.info()
        n_owned = inf["n_owned"]
        self._need_shape(avgs, (n_owned + inf["n_ghost"], self.V), "avgs")
        if out is None:
            out = torch.empty((n_owned, self.V, self.nm), dtype=torch.float64, device=avgs.device)
        if not (out.is_cuda and out.dtype == torch.float64 and out.device == avgs.device):
            raise ValueError("out must be a float64 tensor on the device of avgs")
        self._need_shape(out, (n_owned, self.V, self.nm), "out")
        a_cs, a_vs = avgs.stride()
        c_cs, c_vs, c_ls = out.stride()
        if c_ls != 1:
            raise ValueError("out must be contiguous along the mode axis")
        _check(lib.cwreco_reconstruct(self._h, ctypes.c_void_p(avgs.data_ptr()), a_cs, a_vs,
                                      ctypes.c_void_p(out.data_ptr()), c_cs, c_vs, int(part),
                                      _stream_handle(stream)))
        return out

    def reconstruct_host(self, avgs, out=None, n_pieces=0, stream=None):
        """End to end on HOST buffers (cwreco_reconstruct_host): avgs float64 CPU tensor
        or numpy array [n_local, V] (C-contiguous; page-locked for async copies);
        returns / fills out [n_owned, V, ℳ] on the host.  Synchronous."""
        import torch
        if isinstance(avgs, np.ndarray):
            avgs = torch.from_numpy(np.ascontiguousarray(avgs, dtype=np.float64))
        if avgs.is_cuda or avgs.dtype != torch.float64 or avgs.dim() != 2 or not avgs.is_contiguous():
            raise ValueError("avgs must be a C-contiguous 2-D float64 host tensor")
        inf = self.info()
        self._need_shape(avgs, (inf["n_owned"] + inf["n_ghost"], self.V), "avgs")
        if out is None:
            out = torch.empty((inf["n_owned"], self.V, self.nm), dtype=torch.float64,
                              pin_memory=avgs.is_pinned())
        if out.is_cuda or out.dtype != torch.float64 or not out.is_contiguous():
            raise ValueError("out must be a C-contiguous float64 host tensor")
        self._need_shape(out, (inf["n_owned"], self.V, self.nm), "out")
        _check(lib.cwreco_reconstruct_host(self._h, ctypes.c_void_p(avgs.data_ptr()),
                                           ctypes.c_void_p(out.data_ptr()), int(n_pieces),
                                           _stream_handle(stream)))
        return out

    # ---------------------------------------------------------------- face traces (NEXT-3)
    def face_rule(self):
        """(lam [nq][dim] barycentric weights over the sorted face vertices, weights [nq])."""
        nq = ctypes.c_int()
        _check(lib.cwreco_face_rule(self._h, ctypes.byref(nq), None, None))
        lam = np.empty((nq.value, self.dim))
        w = np.empty(nq.value)
        _check(lib.cwreco_face_rule(self._h, ctypes.byref(nq), _ptr(lam), _ptr(w)))
        return lam, w

    def face_neighbors(self):
        out = np.empty((self.info()["n_owned"], self.dim + 1), dtype=np.int64)
        _check(lib.cwreco_face_neighbors(self._h, _ptr(out)))
        return out

    def face_traces(self, coeffs, out=None, stream=None):
        """coeffs: CUDA [n_owned, V, ℳ] (cwreco_reconstruct output); returns / fills
        out [n_owned, dim+1, nq, V] on the device."""
        import torch
        nq = self.face_rule()[1].shape[0]
        n_owned = self.info()["n_owned"]
        if not (coeffs.is_cuda and coeffs.dtype == torch.float64 and coeffs.dim() == 3):
            raise ValueError("coeffs must be a 3-D float64 CUDA tensor")
        if coeffs.shape[0] < n_owned or tuple(coeffs.shape[1:]) != (self.V, self.nm):
            raise ValueError(f"coeffs must have shape (>= {n_owned}, {self.V}, {self.nm})")
        if out is None:
            out = torch.empty((n_owned, self.dim + 1, nq, self.V), dtype=torch.float64,
                              device=coeffs.device)
        if not (out.is_cuda and out.dtype == torch.float64 and out.device == coeffs.device):
            raise ValueError("out must be a float64 tensor on the device of coeffs")
        self._need_shape(out, (n_owned, self.dim + 1, nq, self.V), "out")
        c_cs, c_vs, c_ls = coeffs.stride()
        if c_ls != 1 or not out.is_contiguous():
            raise ValueError("coeffs must be contiguous along the mode axis and out dense")
        _check(lib.cwreco_face_traces(self._h, ctypes.c_void_p(coeffs.data_ptr()), c_cs, c_vs,
                                      ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    # ---------------------------------------------------------------- predictor (NEXT-2)
    def predictor_setup(self, gamma=1.4):
        """cwreco_predictor_setup: Euler (nvars = dim + 2), after build_stencils."""
        _check(lib.cwreco_predictor_setup(self._h, float(gamma)))

    def predictor_nodes(self):
        """(nodes [𝓛][dim+1] (ξ, τ) in output order, number of known τ = 0 nodes)."""
        # the nodes depend only on (dim, M), fixed for the context; the library rebuilds its
        # host matrices on every query, so predict() must not ask per call
        cached = getattr(self, "_pred_nodes", None)
        if cached is None:
            n, k = ctypes.c_int(), ctypes.c_int()
            _check(lib.cwreco_predictor_nodes(self._h, ctypes.byref(n), ctypes.byref(k), None))
            nodes = np.empty((n.value, self.dim + 1))
            _check(lib.cwreco_predictor_nodes(self._h, ctypes.byref(n), ctypes.byref(k), _ptr(nodes)))
            cached = self._pred_nodes = (nodes, k.value)
        return cached[0].copy(), cached[1]

    def predict(self, coeffs, dt, out=None, iters=None, stream=None):
        """cwreco_predict: coeffs CUDA [n_owned, V, ℳ] (mode axis contiguous) → out
        [n_owned, 𝓛, V] nodal space-time DOFs; iters (optional int32 [n_owned])."""
        import torch
        n_owned = self.info()["n_owned"]
        if not (coeffs.is_cuda and coeffs.dtype == torch.float64 and coeffs.dim() == 3):
            raise ValueError("coeffs must be a 3-D float64 CUDA tensor")
        if coeffs.shape[0] < n_owned or tuple(coeffs.shape[1:]) != (self.V, self.nm) or coeffs.stride(2) != 1:
            raise ValueError(f"coeffs must be (>= {n_owned}, {self.V}, {self.nm}) with contiguous modes")
        L = self.predictor_nodes()[0].shape[0]
        if out is None:
            out = torch.empty((n_owned, L, self.V), dtype=torch.float64, device=coeffs.device)
        if not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()):
            raise ValueError("out must be a dense float64 CUDA tensor")
        self._need_shape(out, (n_owned, L, self.V), "out")
        if iters is not None and (iters.dtype != torch.int32 or tuple(iters.shape) != (n_owned,)):
            raise ValueError("iters must be int32 [n_owned]")
        c_cs, c_vs, _ = coeffs.stride()
        _check(lib.cwreco_predict(self._h, ctypes.c_void_p(coeffs.data_ptr()), c_cs, c_vs, float(dt),
                                  ctypes.c_void_p(out.data_ptr()),
                                  None if iters is None else ctypes.c_void_p(iters.data_ptr()),
                                  _stream_handle(stream)))
        return out

    def reconstruct_debug(self, avgs, cells, stream=None):
        cells = np.ascontiguousarray(cells, dtype=np.int64)
        n, V, nm, d = len(cells), self.V, self.nm, self.dim
        popt = np.empty((n, V, nm))
        psec = np.empty((n, d + 1, V, d + 1))
        sig = np.empty((n, d + 2, V))
        om = np.empty((n, d + 2, V))
        w = np.empty((n, V, nm))
        a_cs, a_vs = avgs.stride()
        _check(lib.cwreco_reconstruct_debug(self._h, ctypes.c_void_p(avgs.data_ptr()), a_cs, a_vs, n, _ptr(cells),
                                            _ptr(popt), _ptr(psec), _ptr(sig), _ptr(om), _ptr(w),
                                            _stream_handle(stream)))
        return dict(popt=popt, psec=psec, sigma=sig, omega=om, w=w)


def setup_context(nodes, cells, period, degree_M, nvars, device=0, rank=0, nranks=1, family=-1, max_ctas=0,
                  uid=None, max_tile=0, **params):
    """set_mesh → set_partition → build_stencils → precompute (family / max_ctas:
    cwreco_set_option, see include/cwreco.h)."""
    ctx = Context(nodes.shape[1], degree_M, nvars, device, **params)
    ctx.set_option(OPT_FAMILY, family)
    if max_ctas:
        ctx.set_option(OPT_MAX_CTAS, max_ctas)
    if max_tile:
        ctx.set_option(OPT_MAX_TILE, max_tile)
    ctx.set_mesh(nodes, cells, period)
    if nranks > 1:
        ctx.set_partition(rank, nranks, uid)
    ctx.build_stencils()
    ctx.precompute()
    return ctx

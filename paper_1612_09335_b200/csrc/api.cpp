// extern "C" surface of libcwreco (include/cwreco.h).  Converts exceptions to
// status codes; keeps a thread-local last-error message.
#include <algorithm>
#include <cstring>
#include <string>

#include "internal.hpp"

namespace {

thread_local std::string g_last_error = "no error";

template <class F>
cwreco_status guard(F&& f) {
  try {
    f();
    return CWRECO_OK;
  } catch (const cwr::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return CWRECO_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CWRECO_EINVAL;
  } catch (...) {
    g_last_error = "unknown error";
    return CWRECO_EINVAL;
  }
}

void need(bool cond, cwreco_status s, const char* msg) {
  if (!cond) cwr::fail(s, msg);
}

// Derived device state (face-trace tables, matrix-free arrays) is built from the
// mesh, partition and stencils: drop it whenever one of those changes.
void invalidate_derived(cwreco_ctx* c) {
  cwr::dev_traces_destroy(c);
  cwr::dev_matfree_destroy(c);
  cwr::dev_predictor_destroy(c);
}

// Coefficient rows (c, v) → c·ccs + v·cvs + [0, ℳ) must not overlap: cell-major
// (cvs ≥ ℳ, ccs ≥ V·cvs) or variable-major (ccs ≥ ℳ, cvs ≥ n·ccs).
void need_disjoint_rows(const cwreco_ctx* c, int64_t ccs, int64_t cvs, int64_t n, const char* what) {
  const bool cell_major = cvs >= c->nm && ccs >= (int64_t)c->V * cvs;
  const bool var_major = ccs >= c->nm && (c->V == 1 || cvs >= n * ccs);
  if (!(cell_major || var_major))
    cwr::fail(CWRECO_EINVAL, std::string(what) + ": coefficient strides make rows overlap (need cvs >= n_modes and "
                                                 "ccs >= nvars*cvs, or ccs >= n_modes and cvs >= n_owned*ccs)");
}

void need_device(const cwreco_ctx* c, const char* what) {
  if (c->device < 0 || !c->dev)
    cwr::fail(CWRECO_ECUDA, std::string(what) + ": host-only context (no CUDA device); there is no CPU fallback");
}

}  // namespace

extern "C" {

const char* cwreco_last_error(void) { return g_last_error.c_str(); }

const char* cwreco_version(void) {
#ifdef CWRECO_EXPERIMENTS
  return "cwreco 0.2.0 (sm_100a) +experiments (timing-only switches compiled in; not a product build)";
#else
  return "cwreco 0.2.0 (sm_100a)";
#endif
}

cwreco_status cwreco_create(int dim, int degree_M, int nvars, const cwreco_params* params, int cuda_device,
                            cwreco_ctx** out) {
  return guard([&] {
    need(out != nullptr, CWRECO_EINVAL, "create: out is NULL");
    *out = nullptr;
    need(dim == 2 || dim == 3, CWRECO_EUNSUPPORTED, "create: dim must be 2 or 3");
    need(degree_M >= 1 && degree_M <= (dim == 2 ? 4 : 3), CWRECO_EUNSUPPORTED, "create: degree out of range");
    need(nvars >= 1 && nvars <= 16, CWRECO_EUNSUPPORTED, "create: nvars must be in [1, 16]");
    if (params) {
      need(params->lambda0 > 0 && params->lambda_s > 0 && params->eps > 0 && params->r >= 1 && params->r <= 16,
           CWRECO_EINVAL, "create: lambda0, lambda_s, eps must be > 0 and 1 <= r <= 16");
    }
    auto* c = new cwreco_ctx();
    c->d = dim;
    c->M = degree_M;
    c->V = nvars;
    c->nm = cwr::n_modes(degree_M, dim);
    c->ne = dim * c->nm;
    if (params) c->prm = *params;
    c->device = cuda_device;
    try {
      cwr::dev_create(c);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void cwreco_destroy(cwreco_ctx* ctx) {
  if (!ctx) return;
  try {
    cwr::halo_destroy(ctx);
    cwr::dev_predictor_destroy(ctx);
    cwr::dev_matfree_destroy(ctx);
    cwr::dev_traces_destroy(ctx);
    cwr::dev_destroy(ctx);
  } catch (...) {
  }
  delete ctx;
}

cwreco_status cwreco_get_info(const cwreco_ctx* c, cwreco_info* o) {
  return guard([&] {
    need(c && o, CWRECO_EINVAL, "get_info: NULL");
    std::memset(o, 0, sizeof(*o));
    o->dim = c->d;
    o->degree_M = c->M;
    o->nvars = c->V;
    o->n_modes = c->nm;
    o->n_e = c->ne;
    o->gather_len = c->G;
    o->n_cells = c->N;
    o->n_owned = c->n_owned;
    o->n_ghost = c->n_ghost;
    o->n_interior = c->n_interior;
    o->n_invalid_sectors = c->n_invalid;
    o->n_extra_gather = c->n_extra;
    o->union_max = c->lay.Umax;
    o->kernel_family = c->has_blocks ? c->lay.kind : -1;
    o->n_boundary_ghosts = (int64_t)c->bc_ids.size();
    if (c->has_blocks) {
      o->tile_cells = c->lay.T;
      o->chunk_k = c->lay.KC;
      o->n_tiles = c->n_tiles;
      o->n_interior_tiles = c->n_int_tiles;
      o->tile_bytes = c->lay.tile_bytes;
    }
    o->device_bytes = cwr::dev_bytes(c);
    const int d = c->d, nm = c->nm, ne = c->ne, V = c->V;
    // 8[(ℳ-1)(n_e-1) + (d+1)d²] + 4(n_e-1) + (d+1)d + 8V + 8ℳV
    o->algorithmic_bytes_per_cell =
        8LL * ((nm - 1) * (ne - 1) + (d + 1) * d * d) + 4LL * (ne - 1) + (d + 1) * d + 8LL * V + 8LL * nm * V;
  });
}

cwreco_status cwreco_set_kernel(cwreco_ctx* c, int variant) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "set_kernel: NULL");
    need(variant == CWRECO_KERNEL_PIPELINED || variant == CWRECO_KERNEL_SIMPLE ||
             variant == CWRECO_KERNEL_MATRIXFREE,
         CWRECO_EINVAL, "set_kernel: unknown variant");
    c->kernel = variant;
  });
}

cwreco_status cwreco_set_option(cwreco_ctx* c, int option, int64_t value) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "set_option: NULL");
    switch (option) {
      case CWRECO_OPT_FAMILY:
        need(value >= -1 && value <= 1, CWRECO_EINVAL, "set_option: family must be -1, 0 or 1");
        c->family = (int)value;
        c->has_blocks = false;  // the packed layout depends on the family
        break;
      case CWRECO_OPT_MAX_CTAS:
        need(value >= 0 && value <= (1 << 30), CWRECO_EINVAL, "set_option: max_ctas must be >= 0");
        c->max_ctas = value;
        break;
      case CWRECO_OPT_MAX_TILE:
        need(value >= 0 && value <= (1 << 16), CWRECO_EINVAL, "set_option: max_tile must be >= 0");
        c->max_tile = value;
        c->has_blocks = false;  // the packed layout depends on the tile size
        break;
      default:
        cwr::fail(CWRECO_EINVAL, "set_option: unknown option " + std::to_string(option));
    }
  });
}

cwreco_status cwreco_set_mesh(cwreco_ctx* c, int64_t n_nodes, const double* xyz, int64_t n_cells,
                              const int64_t* cell_nodes, const double* period) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "set_mesh: NULL ctx");
    invalidate_derived(c);
    cwr::set_mesh(c, n_nodes, xyz, n_cells, cell_nodes, period);
  });
}

cwreco_status cwreco_set_boundary(cwreco_ctx* c, const int* side_bc, int mom0) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "set_boundary: NULL ctx");
    need(c->has_mesh, CWRECO_ESTATE, "set_boundary: call cwreco_set_mesh first");
    need(!c->periodic, CWRECO_EINVAL, "set_boundary: boundary ghost cells need an open mesh (period = NULL)");
    need(mom0 >= -1 && mom0 + c->d <= c->V, CWRECO_EINVAL, "set_boundary: mom0 must be -1 or leave room for dim momenta");
    bool any = false;
    for (int s = 0; s < 2 * c->d; ++s) {
      const int b = side_bc ? side_bc[s] : 0;
      need(b >= 0 && b <= 2, CWRECO_EINVAL, "set_boundary: side codes are 0 (none), 1 (transmissive), 2 (wall)");
      any |= b != 0;
    }
    need(!any || c->N * int64_t(2 * c->d + 1) < INT32_MAX, CWRECO_EUNSUPPORTED,
         "set_boundary: ghost ids exceed 32 bits");
    invalidate_derived(c);
    for (int s = 0; s < 6; ++s) c->bc[s] = (side_bc && s < 2 * c->d) ? side_bc[s] : 0;
    c->mom0 = mom0;
    c->has_bc = any;
    c->bc_ids.clear();
    c->has_stencils = c->has_blocks = false;
  });
}

cwreco_status cwreco_get_permutation(const cwreco_ctx* c, int64_t* out) {
  return guard([&] {
    need(c && out, CWRECO_EINVAL, "get_permutation: NULL");
    need(c->has_mesh, CWRECO_ESTATE, "get_permutation: no mesh");
    std::memcpy(out, c->perm.data(), sizeof(int64_t) * c->N);
  });
}

cwreco_status cwreco_set_partition(cwreco_ctx* c, int rank, int nranks, const uint8_t* id) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "set_partition: NULL");
    need(nranks >= 1 && rank >= 0 && rank < nranks, CWRECO_EINVAL, "set_partition: bad rank/nranks");
    invalidate_derived(c);
    cwr::halo_destroy(c);
    c->rank = rank;
    c->nranks = nranks;
    c->has_stencils = c->has_blocks = false;
    if (c->has_mesh) {
      c->own_lo = (rank * c->N) / nranks;
      c->own_hi = ((rank + 1) * c->N) / nranks;
    }
    cwr::halo_set_transport(c, id);
  });
}

cwreco_status cwreco_nccl_unique_id(uint8_t* id) {
  return guard([&] {
    need(id != nullptr, CWRECO_EINVAL, "nccl_unique_id: NULL");
    cwr::halo_unique_id_nccl(id);
  });
}

cwreco_status cwreco_loopback_unique_id(int nranks, uint8_t* id) {
  return guard([&] {
    need(id != nullptr, CWRECO_EINVAL, "loopback_unique_id: NULL");
    cwr::halo_unique_id_loopback(nranks, id);
  });
}

cwreco_status cwreco_build_stencils(cwreco_ctx* c) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "build_stencils: NULL");
    need(c->has_mesh, CWRECO_ESTATE, "build_stencils: call cwreco_set_mesh first");
    need(c->own_hi > c->own_lo, CWRECO_EINVAL, "build_stencils: this rank owns no cells");
    invalidate_derived(c);
    cwr::build_stencils(c);
    cwr::halo_plan_exchange(c);  // collective when a transport is set
  });
}

cwreco_status cwreco_get_stencils(const cwreco_ctx* c, int32_t* central, int32_t* sectors, uint8_t* valid) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "get_stencils: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "get_stencils: no stencils");
    const int ne = c->ne, nv = c->d + 1;
    for (int64_t li = 0; li < c->n_owned; ++li) {
      const int64_t q = c->local2global[li] - c->own_lo;
      if (central) std::memcpy(central + li * ne, &c->central[q * ne], sizeof(int32_t) * ne);
      if (sectors) std::memcpy(sectors + li * nv * nv, &c->sectors[q * nv * nv], sizeof(int32_t) * nv * nv);
      if (valid) std::memcpy(valid + li * nv, &c->valid[q * nv], nv);
    }
  });
}

cwreco_status cwreco_prepare_matrixfree(cwreco_ctx* c) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "prepare_matrixfree: NULL ctx");
    need_device(c, "prepare_matrixfree");
    cwr::MatfreeHost h;
    cwr::matfree_prepare(c, h);
    cwr::dev_matfree_upload(c, h);
  });
}

cwreco_status cwreco_set_stencils(cwreco_ctx* c, const int32_t* central, const int32_t* sectors,
                                  const uint8_t* valid) {
  return guard([&] {
    need(c && central && sectors && valid, CWRECO_EINVAL, "set_stencils: NULL");
    need(c->has_mesh, CWRECO_ESTATE, "set_stencils: no mesh");
    const int ne = c->ne, nv = c->d + 1;
    const int64_t lo = c->own_lo, n_own = c->own_hi - c->own_lo;
    for (int64_t q = 0; q < n_own; ++q) {
      const int64_t i = lo + q;
      const int32_t* cen = central + q * ne;
      if (cen[0] != i)
        cwr::fail(CWRECO_EINVAL, "set_stencils: central stencil of cell " + std::to_string(i) +
                                     " must start with the cell itself");
      for (int k = 0; k < ne; ++k) {
        need(cen[k] >= 0 && cen[k] < c->N, CWRECO_EINVAL, "set_stencils: cell id out of range");
        for (int m = 0; m < k; ++m) need(cen[m] != cen[k], CWRECO_EINVAL, "set_stencils: repeated cell in a stencil");
      }
      for (int v = 0; v < nv; ++v) {
        need(valid[q * nv + v] <= 1, CWRECO_EINVAL, "set_stencils: valid flags must be 0 or 1");
        const int32_t* sec = sectors + (q * nv + v) * nv;
        if (!valid[q * nv + v]) continue;
        need(sec[0] == i, CWRECO_EINVAL, "set_stencils: a valid sector must start with the cell itself");
        for (int k = 1; k < nv; ++k) {
          need(sec[k] >= 0 && sec[k] < c->N && sec[k] != i, CWRECO_EINVAL, "set_stencils: bad sector member");
          for (int m = 1; m < k; ++m) need(sec[m] != sec[k], CWRECO_EINVAL, "set_stencils: repeated sector member");
        }
      }
    }
    c->central.assign(central, central + n_own * ne);
    c->sectors.assign(sectors, sectors + n_own * nv * nv);
    c->valid.assign(valid, valid + n_own * nv);
    for (int64_t q = 0; q < n_own; ++q)  // invalid sectors carry no members
      for (int v = 0; v < nv; ++v)
        if (!c->valid[q * nv + v])
          for (int k = 0; k < nv; ++k) c->sectors[(q * nv + v) * nv + k] = -1;
    invalidate_derived(c);
    cwr::finalize_stencils(c);
    cwr::halo_plan_exchange(c);  // collective when a transport is set
  });
}

cwreco_status cwreco_get_local_cells(const cwreco_ctx* c, int64_t* out) {
  return guard([&] {
    need(c && out, CWRECO_EINVAL, "get_local_cells: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "get_local_cells: no stencils");
    std::memcpy(out, c->local2global.data(), sizeof(int64_t) * c->local2global.size());
  });
}

cwreco_status cwreco_precompute(cwreco_ctx* c) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "precompute: NULL");
    cwr::precompute(c);
  });
}

cwreco_status cwreco_get_sigma(const cwreco_ctx* c, double* out) {
  return guard([&] {
    need(c && out, CWRECO_EINVAL, "get_sigma: NULL");
    std::vector<double> S = c->sigma.empty() ? cwr::sigma_matrix(c->d, c->M) : c->sigma;
    std::memcpy(out, S.data(), sizeof(double) * S.size());
  });
}

cwreco_status cwreco_get_blocks(const cwreco_ctx* c, int64_t n_sel, const int64_t* cells, double* bplus, double* sinv,
                                int32_t* gather, uint8_t* slots) {
  return guard([&] {
    need(c && (n_sel == 0 || cells), CWRECO_EINVAL, "get_blocks: NULL");
    need(c->has_blocks, CWRECO_ESTATE, "get_blocks: call cwreco_precompute first");
    const cwr::Layout& L = c->lay;
    const int T = L.T, R = L.R, G = L.G, d = c->d, nv = d + 1;
    std::vector<unsigned char> tile(L.tile_bytes);
    int64_t cur = -1;
    for (int64_t s = 0; s < n_sel; ++s) {
      const int64_t li = cells[s];
      need(li >= 0 && li < c->n_owned, CWRECO_EINVAL, "get_blocks: cell out of range");
      const int64_t t = li / T;
      const int ct = int(li % T);
      const unsigned char* tb;
      if (!c->host_blocks.empty()) {
        tb = c->host_blocks.data() + t * L.tile_bytes;
      } else {
        if (t != cur) {
          cwr::dev_download_tile(c, t, tile.data());
          cur = t;
        }
        tb = tile.data();
      }
      const double* sv = (const double*)(tb + cwr::sector_sinv_off(L.off_sector, L.sector_bytes, L.TSC, L.srec, ct));
      const uint8_t vm = *(tb + cwr::sector_mask_off(L.off_sector, L.sector_bytes, L.sinv_bytes, L.TSC, ct));
      if (bplus)
        for (int l = 0; l < R; ++l)
          for (int k = 0; k < G; ++k) {
            const int ch = k / L.KC, kk = k % L.KC, kc = L.kc_of(ch);
            const double* B = (const double*)(tb + L.off_chunk(ch) + L.ids_bytes);
            bplus[(s * R + l) * G + k] = B[cwr::chunk_elem(L.kind, kc, R, L.V, T, l, ct, kk)];
          }
      if (sinv) std::memcpy(sinv + s * nv * d * d, sv, sizeof(double) * nv * d * d);
      if (gather)
        for (int k = 0; k < G; ++k) {
          const uint16_t u = ((const uint16_t*)(tb + L.off_idx))[cwr::idx_elem(L.kind, T, k, ct)];
          gather[s * G + k] = ((const int32_t*)tb)[u / L.VP];  // union chunk: local ids
        }
      if (slots)
        for (int q = 0; q < nv; ++q)
          for (int m = 0; m < d; ++m) slots[(s * nv + q) * d + m] = ((vm >> q) & 1) ? uint8_t(q * d + m) : 255;
    }
  });
}

cwreco_status cwreco_halo_plan(const cwreco_ctx* c, int64_t* recv_counts, int64_t* recv_ids) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "halo_plan: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "halo_plan: no stencils");
    if (recv_counts) std::memcpy(recv_counts, c->ghost_counts.data(), sizeof(int64_t) * c->nranks);
    if (recv_ids)
      std::memcpy(recv_ids, c->local2global.data() + c->n_owned, sizeof(int64_t) * c->n_ghost);
  });
}

cwreco_status cwreco_set_send_lists(cwreco_ctx* c, const int64_t* send_counts, const int64_t* send_ids) {
  return guard([&] {
    need(c && send_counts, CWRECO_EINVAL, "set_send_lists: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "set_send_lists: no stencils");
    cwr::install_send_lists(c, send_counts, send_ids);
  });
}

cwreco_status cwreco_get_send_lists(const cwreco_ctx* c, int64_t* send_counts, int64_t* send_ids) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "get_send_lists: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "get_send_lists: no stencils");
    if (send_counts)
      for (int r = 0; r < c->nranks; ++r) send_counts[r] = r < (int)c->send_counts.size() ? c->send_counts[r] : 0;
    if (send_ids)
      for (size_t k = 0; k < c->send_local.size(); ++k) send_ids[k] = c->local2global[c->send_local[k]];
  });
}

cwreco_status cwreco_send_total(const cwreco_ctx* c, int64_t* total) {
  return guard([&] {
    need(c && total, CWRECO_EINVAL, "send_total: NULL");
    *total = (int64_t)c->send_local.size();
  });
}

cwreco_status cwreco_halo_pack(cwreco_ctx* c, const double* d_avgs, int64_t acs, int64_t avs, double* d_sendbuf,
                               cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "halo_pack: NULL");
    need_device(c, "halo_pack");
    if (c->send_local.empty()) return;
    need(d_avgs && d_sendbuf, CWRECO_EINVAL, "halo_pack: NULL buffer");
    cwr::dev_halo_pack(c, d_avgs, acs, avs, d_sendbuf, stream);
  });
}

cwreco_status cwreco_halo_pack_rows(cwreco_ctx* c, const double* d_rows, int64_t row_stride, int width,
                                    double* d_sendbuf, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "halo_pack_rows: NULL");
    need_device(c, "halo_pack_rows");
    need(width >= 1 && row_stride >= width, CWRECO_EINVAL, "halo_pack_rows: bad width / stride");
    if (c->send_local.empty()) return;
    need(d_rows && d_sendbuf, CWRECO_EINVAL, "halo_pack_rows: NULL buffer");
    cwr::dev_halo_pack_rows(c, d_rows, row_stride, 1, width, d_sendbuf, stream);
  });
}

cwreco_status cwreco_reconstruct(cwreco_ctx* c, const double* d_avgs, int64_t acs, int64_t avs, double* d_coeffs,
                                 int64_t ccs, int64_t cvs, int part, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "reconstruct: NULL ctx");
    need_device(c, "reconstruct");
    if (c->kernel == CWRECO_KERNEL_MATRIXFREE)
      need(c->mf != nullptr, CWRECO_ESTATE, "reconstruct: call cwreco_prepare_matrixfree first");
    else
      need(c->has_blocks, CWRECO_ESTATE, "reconstruct: call cwreco_precompute first");
    need(d_avgs && d_coeffs, CWRECO_EINVAL, "reconstruct: NULL buffer");
    need(acs >= 1 && avs >= 1 && ccs >= 1 && cvs >= 1, CWRECO_EINVAL, "reconstruct: strides must be >= 1");
    need_disjoint_rows(c, ccs, cvs, c->n_owned, "reconstruct");
    need(part == CWRECO_PART_ALL || part == CWRECO_PART_INTERIOR || part == CWRECO_PART_BOUNDARY, CWRECO_EINVAL,
         "reconstruct: bad part");
    cwr::dev_reconstruct(c, d_avgs, acs, avs, d_coeffs, ccs, cvs, part, stream);
  });
}

cwreco_status cwreco_halo_exchange(cwreco_ctx* c, double* d_avgs, int64_t acs, int64_t avs, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "halo_exchange: NULL ctx");
    need_device(c, "halo_exchange");
    need(c->has_stencils, CWRECO_ESTATE, "halo_exchange: no stencils");
    need(d_avgs != nullptr, CWRECO_EINVAL, "halo_exchange: NULL buffer");
    need(acs >= 1 && avs >= 1, CWRECO_EINVAL, "halo_exchange: strides must be >= 1");
    if (c->nranks == 1) return;
    cwr::halo_exchange(c, d_avgs, acs, avs, c->V, stream);
  });
}

cwreco_status cwreco_halo_exchange_rows(cwreco_ctx* c, double* d_rows, int64_t row_stride, int width,
                                        cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "halo_exchange_rows: NULL ctx");
    need_device(c, "halo_exchange_rows");
    need(c->has_stencils, CWRECO_ESTATE, "halo_exchange_rows: no stencils");
    need(d_rows != nullptr, CWRECO_EINVAL, "halo_exchange_rows: NULL buffer");
    need(width >= 1 && row_stride >= width, CWRECO_EINVAL, "halo_exchange_rows: bad width / stride");
    if (c->nranks == 1) return;
    cwr::halo_exchange(c, d_rows, row_stride, 1, width, stream);
  });
}

cwreco_status cwreco_reconstruct_overlap(cwreco_ctx* c, double* d_avgs, int64_t acs, int64_t avs, double* d_coeffs,
                                         int64_t ccs, int64_t cvs, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "reconstruct_overlap: NULL ctx");
    need_device(c, "reconstruct_overlap");
    if (c->kernel == CWRECO_KERNEL_MATRIXFREE)
      need(c->mf != nullptr, CWRECO_ESTATE, "reconstruct_overlap: call cwreco_prepare_matrixfree first");
    else
      need(c->has_blocks, CWRECO_ESTATE, "reconstruct_overlap: call cwreco_precompute first");
    need(d_avgs && d_coeffs, CWRECO_EINVAL, "reconstruct_overlap: NULL buffer");
    need(acs >= 1 && avs >= 1 && ccs >= 1 && cvs >= 1, CWRECO_EINVAL, "reconstruct_overlap: strides must be >= 1");
    need_disjoint_rows(c, ccs, cvs, c->n_owned, "reconstruct_overlap");
    if (c->nranks == 1) {
      cwr::dev_reconstruct(c, d_avgs, acs, avs, d_coeffs, ccs, cvs, CWRECO_PART_ALL, stream);
      return;
    }
    cwr::halo_reconstruct_overlap(c, d_avgs, acs, avs, d_coeffs, ccs, cvs, stream);
  });
}

cwreco_status cwreco_reconstruct_host(cwreco_ctx* c, const double* h_avgs, double* h_coeffs, int n_pieces,
                                      cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "reconstruct_host: NULL ctx");
    need_device(c, "reconstruct_host");
    if (c->kernel == CWRECO_KERNEL_MATRIXFREE)
      need(c->mf != nullptr, CWRECO_ESTATE, "reconstruct_host: call cwreco_prepare_matrixfree first");
    else
      need(c->has_blocks, CWRECO_ESTATE, "reconstruct_host: call cwreco_precompute first");
    need(h_avgs && h_coeffs, CWRECO_EINVAL, "reconstruct_host: NULL buffer");
    cwr::dev_reconstruct_host(c, h_avgs, h_coeffs, n_pieces > 0 ? n_pieces : 4, stream);
  });
}

cwreco_status cwreco_predictor_setup(cwreco_ctx* c, double gamma) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "predictor_setup: NULL ctx");
    need_device(c, "predictor_setup");
    need(c->has_stencils, CWRECO_ESTATE, "predictor_setup: call cwreco_build_stencils first (local numbering)");
    need(c->M <= 3, CWRECO_EUNSUPPORTED, "predictor_setup: degree M must be <= 3");
    need(c->V == c->d + 2, CWRECO_EUNSUPPORTED, "predictor_setup: the Euler system needs nvars = dim + 2");
    need(gamma > 1.0, CWRECO_EINVAL, "predictor_setup: gamma must be > 1");
    cwr::PredictorHost h;
    cwr::predictor_matrices(c->d, c->M, h);
    std::vector<double> jinv;
    cwr::predictor_jinv(c, jinv);
    cwr::dev_predictor_setup(c, h, jinv, gamma);
  });
}

cwreco_status cwreco_predictor_nodes(const cwreco_ctx* c, int* n_nodes, int* n_known, double* nodes) {
  return guard([&] {
    need(c && n_nodes && n_known, CWRECO_EINVAL, "predictor_nodes: NULL");
    need(c->M <= 3, CWRECO_EUNSUPPORTED, "predictor_nodes: degree M must be <= 3");
    cwr::PredictorHost h;
    cwr::predictor_matrices(c->d, c->M, h);
    *n_nodes = h.L;
    *n_known = h.nk;
    if (nodes) std::memcpy(nodes, h.nodes.data(), sizeof(double) * h.nodes.size());
  });
}

cwreco_status cwreco_predict(cwreco_ctx* c, const double* d_coeffs, int64_t ccs, int64_t cvs, double dt,
                             double* d_qhat, int32_t* d_iters, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "predict: NULL ctx");
    need_device(c, "predict");
    need(c->pred != nullptr, CWRECO_ESTATE, "predict: call cwreco_predictor_setup first");
    need(d_coeffs && d_qhat, CWRECO_EINVAL, "predict: NULL buffer");
    need(ccs >= 1 && cvs >= 1, CWRECO_EINVAL, "predict: strides must be >= 1");
    need(dt >= 0.0, CWRECO_EINVAL, "predict: dt must be >= 0");
    cwr::dev_predict(c, d_coeffs, ccs, cvs, dt, d_qhat, d_iters, stream);
  });
}

cwreco_status cwreco_face_rule(const cwreco_ctx* c, int* nq, double* lam, double* weights) {
  return guard([&] {
    need(c && nq, CWRECO_EINVAL, "face_rule: NULL");
    std::vector<double> l, w;
    cwr::face_rule(c->d, c->M, l, w);
    *nq = (int)w.size();
    if (lam) std::memcpy(lam, l.data(), sizeof(double) * l.size());
    if (weights) std::memcpy(weights, w.data(), sizeof(double) * w.size());
  });
}

cwreco_status cwreco_face_neighbors(const cwreco_ctx* c, int64_t* nbr) {
  return guard([&] {
    need(c && nbr, CWRECO_EINVAL, "face_neighbors: NULL");
    need(c->has_stencils, CWRECO_ESTATE, "face_neighbors: no stencils");
    const int nv = c->d + 1;
    const int64_t n_loc = c->n_owned + c->n_ghost;
    std::vector<int64_t> sorted_ids(c->local2global.begin(), c->local2global.begin() + n_loc);
    std::vector<int64_t> order(n_loc);
    for (int64_t k = 0; k < n_loc; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sorted_ids[a] < sorted_ids[b]; });
    std::vector<int64_t> keys(n_loc);
    for (int64_t k = 0; k < n_loc; ++k) keys[k] = sorted_ids[order[k]];
    for (int64_t li = 0; li < c->n_owned; ++li) {
      const int64_t g = c->local2global[li];
      for (int f = 0; f < nv; ++f) {
        const int64_t j = c->nbr[g * nv + f];
        int64_t lj = -1;
        if (j >= 0) {
          auto it = std::lower_bound(keys.begin(), keys.end(), j);
          need(it != keys.end() && *it == j, CWRECO_EINVAL, "face_neighbors: neighbour not local");
          lj = order[it - keys.begin()];
        }
        nbr[li * nv + f] = lj;
      }
    }
  });
}

cwreco_status cwreco_face_traces(cwreco_ctx* c, const double* d_coeffs, int64_t ccs, int64_t cvs, double* d_traces,
                                 cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "face_traces: NULL ctx");
    need_device(c, "face_traces");
    need(c->has_stencils, CWRECO_ESTATE, "face_traces: no stencils");
    need(d_coeffs && d_traces, CWRECO_EINVAL, "face_traces: NULL buffer");
    need_disjoint_rows(c, ccs, cvs, c->n_owned, "face_traces");
    cwr::dev_face_traces(c, d_coeffs, ccs, cvs, d_traces, stream);
  });
}

cwreco_status cwreco_reconstruct_debug(cwreco_ctx* c, const double* d_avgs, int64_t acs, int64_t avs, int64_t n_sel,
                                       const int64_t* cells, double* popt, double* psec, double* sigma,
                                       double* omega, double* w, cwreco_stream stream) {
  return guard([&] {
    need(c != nullptr, CWRECO_EINVAL, "reconstruct_debug: NULL ctx");
    need_device(c, "reconstruct_debug");
    need(c->has_blocks, CWRECO_ESTATE, "reconstruct_debug: call cwreco_precompute first");
    need(d_avgs && (n_sel == 0 || cells), CWRECO_EINVAL, "reconstruct_debug: NULL");
    for (int64_t s = 0; s < n_sel; ++s)
      need(cells[s] >= 0 && cells[s] < c->n_owned, CWRECO_EINVAL, "reconstruct_debug: cell out of range");
    if (n_sel == 0) return;
    cwr::dev_debug(c, d_avgs, acs, avs, n_sel, cells, popt, psec, sigma, omega, w, stream);
  });
}

}  // extern "C"
